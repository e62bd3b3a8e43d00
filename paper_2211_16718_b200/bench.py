"""Memory-layout / traversal study of the nonlinear-weight kernel on the GPU.

The reference's microbenchmark (pkg/src/hitdns/bench.py, kernels.py:236-329)
asks how the data layout and the visiting order change the throughput of the
WENO weight computation; here the kernel is ``hd_bench_weights`` in libhd.so
and every repeat is timed with CUDA events on the launching stream:

* layout: INTERLEAVED (AoS: the five variables of a point adjacent) or
  COMPONENT_CONTIGUOUS (SoA: one variable's points adjacent);
* traversal ``"lex"``: one thread per active point, x fastest (SoA: a warp
  reads 256 contiguous bytes per load; AoS: a 40-byte stride, 5x the sectors);
  ``"tiled"``: (tx, ty) thread tiles over each z plane, whose lanes past a
  ragged edge idle (the reference's wasted iterations).

Public names and numbers follow the reference (X_PAD, BYTES_PER_POINT = 320,
the seeded dataset, the report's columns, the soft ordering warnings) so its
tests and reports carry over; the weights themselves are bitwise the
reference's for every layout x traversal (tests/golden/bench_weights.npz).
"""

from __future__ import annotations

import ctypes
import warnings
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .grid import Layout
from .physics import DEFAULT_PARAMS, WenoParams

NVARS = 5
X_PAD = 2                           # x reach of the 5-point stencil
BYTES_PER_POINT = NVARS * 8 * (5 + 3)  # per active point: 5 stencil reads + 3 weight writes per variable
DEFAULT_SIZES = (16, 32, 48, 64)
DEFAULT_TILE = (32, 8)
TRAVERSALS = ("lex", "tiled")
BENCH_SEED = 20170907
_LAYOUT_LABEL = {Layout.INTERLEAVED: "interleaved", Layout.COMPONENT_CONTIGUOUS: "contiguous"}


def _extents(n) -> tuple:
    """(nx, ny, nz) from a cube edge or a triple."""
    return (int(n),) * 3 if np.isscalar(n) else tuple(int(v) for v in n)


def _padded_points(nx: int, ny: int, nz: int) -> int:
    return (nx + 2 * X_PAD) * ny * nz


def make_bench_values(shape, seed: int = BENCH_SEED) -> np.ndarray:
    """The seeded dataset, (padded points, 5) values in [0.5, 1.5) so the weights
    stay well conditioned (bench.py:45-50: one default_rng draw)."""
    rng = np.random.default_rng(seed)
    return rng.random((_padded_points(*_extents(shape)), NVARS)) + 0.5


def pack_values(values: np.ndarray, layout: Layout) -> np.ndarray:
    """The flat buffer of a layout: point-major (AoS) or variable-major (SoA)."""
    table = values if layout == Layout.INTERLEAVED else values.T
    return np.ascontiguousarray(table).ravel()


@dataclass
class BenchRecord:
    """Timings (seconds per repeat) of one shape x layout x traversal."""

    shape: tuple
    layout: Layout
    traversal: str
    times: list = field(default_factory=list)
    wasted_lanes: int = 0

    def _t(self) -> np.ndarray:
        return np.asarray(self.times, dtype=np.float64)

    @property
    def active_points(self) -> int:
        return int(np.prod(self.shape))

    @property
    def median_seconds(self) -> float:
        return float(np.median(self._t()))

    @property
    def min_seconds(self) -> float:
        return float(self._t().min())

    @property
    def cv(self) -> float:
        """Coefficient of variation (population std / mean) of the repeats."""
        t = self._t()
        return float(t.std() / t.mean()) if t.mean() > 0.0 else 0.0

    @property
    def bandwidth_gbs(self) -> float:
        return self.active_points * BYTES_PER_POINT / self.median_seconds * 1e-9

    @property
    def wasted_fraction(self) -> float:
        total = self.active_points + self.wasted_lanes
        return self.wasted_lanes / total if total else 0.0

    @property
    def size_label(self) -> str:
        nx, ny, nz = self.shape
        return f"{nx}" if nx == ny == nz else f"{nx}x{ny}x{nz}"


def _layout_name(layout: Layout) -> str:
    return _LAYOUT_LABEL[Layout(layout)]


class _WeightKernel:
    """hd_bench_weights bound to one device dataset and output buffer."""

    def __init__(self, shape, layout: Layout, traversal: str, tile, params: WenoParams, seed: int):
        self.L = _lib.load(require_cuda=True)
        self.shape = shape
        self.layout = Layout(layout)
        self.code = TRAVERSALS.index(traversal)
        self.tile = (int(tile[0]), int(tile[1]))
        self.params = params
        self.data = torch.from_numpy(pack_values(make_bench_values(shape, seed), self.layout)).cuda()
        self.out = torch.zeros(3 * NVARS * _padded_points(*shape), dtype=torch.float64, device="cuda")
        self.wasted = ctypes.c_int64(0)
        self.stream = torch.cuda.current_stream()

    def launch(self) -> None:
        nx, ny, nz = self.shape
        status = self.L.hd_bench_weights(
            self.data.data_ptr(), int(self.layout), self.code, nx, ny, nz, X_PAD, *self.tile,
            float(self.params.epsilon), int(self.params.power), self.out.data_ptr(),
            ctypes.byref(self.wasted), ctypes.c_void_p(self.stream.cuda_stream))
        _lib.check(status, "hd_bench_weights")

    def timed(self) -> float:
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        start.record(self.stream)
        self.launch()
        stop.record(self.stream)
        stop.synchronize()
        return start.elapsed_time(stop) * 1e-3


def run_case(shape, layout: Layout, traversal: str = "lex", repeats: int = 5,
             tile: tuple = DEFAULT_TILE, params: WenoParams = DEFAULT_PARAMS,
             seed: int = BENCH_SEED) -> tuple:
    """One configuration on the current device: (record, point-major weights).
    One untimed launch first (module load), then ``repeats`` timed ones."""
    if traversal not in TRAVERSALS:
        raise ValueError(f"traversal must be one of {TRAVERSALS}, got {traversal!r}")
    if repeats < 1:
        raise ValueError("repeats must be at least 1")
    shape = _extents(shape)
    kernel = _WeightKernel(shape, layout, traversal, tile, params, seed)
    kernel.launch()
    times = [kernel.timed() for _ in range(repeats)]
    record = BenchRecord(shape=shape, layout=Layout(layout), traversal=traversal, times=times,
                         wasted_lanes=int(kernel.wasted.value))
    return record, kernel.out.cpu().numpy()


def layout_sweep(sizes=DEFAULT_SIZES, repeats: int = 5, traversals=("lex",),
                 tile: tuple = DEFAULT_TILE) -> list:
    """Records for sizes x (interleaved, contiguous) x traversals, in that nesting."""
    return [run_case(n, layout, trav, repeats=repeats, tile=tile)[0]
            for n in sizes
            for layout in (Layout.INTERLEAVED, Layout.COMPONENT_CONTIGUOUS)
            for trav in traversals]


def bench_report(records: list) -> str:
    """``n layout traversal median_s bandwidth_GBs ratio_vs_baseline`` rows; the
    baseline of a size is its interleaved/lex record when present, else its
    first record; a trailing ``# max_cv`` line (bench.py:163-189)."""
    base = {}
    for rec in records:
        first = rec.size_label not in base
        if first or (rec.layout == Layout.INTERLEAVED and rec.traversal == "lex"):
            base[rec.size_label] = rec.median_seconds
    rows = ["n layout traversal median_s bandwidth_GBs ratio_vs_baseline"]
    rows += [" ".join((r.size_label, _layout_name(r.layout), r.traversal, f"{r.median_seconds:.3g}",
                       f"{r.bandwidth_gbs:.3g}", f"{r.median_seconds / base[r.size_label]:.3g}"))
             for r in records]
    if records:
        rows.append(f"# max_cv {max(r.cv for r in records):.3g}")
    return "\n".join(rows) + "\n"


def soft_ordering_checks(records: list) -> list:
    """Orderings the study expects but cannot guarantee (cache- and
    scheduler-dependent), returned and emitted as RuntimeWarnings: SoA/lex at
    least as fast as AoS/lex; a tiled run that idles lanes no faster than lex."""
    table = {(r.size_label, Layout(r.layout), r.traversal): r for r in records}
    notes = []
    for size in sorted({r.size_label for r in records}):
        aos, soa = table.get((size, Layout.INTERLEAVED, "lex")), table.get((size, Layout.COMPONENT_CONTIGUOUS, "lex"))
        if aos is not None and soa is not None and soa.median_seconds > aos.median_seconds:
            notes.append(f"n={size}: contiguous layout was slower than interleaved "
                         f"({soa.median_seconds:.3g}s vs {aos.median_seconds:.3g}s)")
        for layout in (Layout.INTERLEAVED, Layout.COMPONENT_CONTIGUOUS):
            lex, tiled = table.get((size, layout, "lex")), table.get((size, layout, "tiled"))
            if lex is None or tiled is None or not tiled.wasted_lanes:
                continue
            if tiled.median_seconds < lex.median_seconds:
                notes.append(f"n={size} {_layout_name(layout)}: tiled traversal beat lexicographic "
                             f"despite wasting {tiled.wasted_fraction:.1%} of its lanes")
    for note in notes:
        warnings.warn(note, RuntimeWarning, stacklevel=2)
    return notes
