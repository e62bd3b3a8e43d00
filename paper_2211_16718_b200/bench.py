"""Memory-layout and traversal study of the nonlinear-weight kernel, on the GPU.

Mirrors pkg/src/hitdns/bench.py (X_PAD, BYTES_PER_POINT, DEFAULT_SIZES,
DEFAULT_TILE, TRAVERSALS, BENCH_SEED, make_bench_values, pack_values,
BenchRecord, run_case, layout_sweep, bench_report, soft_ordering_checks) with
the numba kernels (kernels.py:236-329) replaced by ``hd_bench_weights`` in
libhd.so:

* layout: INTERLEAVED (AoS) or COMPONENT_CONTIGUOUS (SoA) device buffers;
* traversal: ``"lex"`` -- one thread per active point, x fastest, so a warp
  reads 32 consecutive points of one variable (SoA: 256 B per load, fully
  coalesced; AoS: stride 40 B, 5x the sectors); ``"tiled"`` -- (tx, ty)
  thread blocks over x-y tiles of each z plane, with idle lanes where the
  tile overhangs a ragged extent (the reference's wasted iterations).

Each repeat is timed with CUDA events on the launching stream; the output is
the same point-major weight array as the reference, bitwise, for every
layout x traversal combination (kernel operations in the reference order,
never contracted).
"""

from __future__ import annotations

import ctypes
import statistics
import warnings
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .grid import Layout
from .physics import DEFAULT_PARAMS, WenoParams

NVARS = 5
X_PAD = 2  # stencil reach of the weight kernel along x
BYTES_PER_POINT = NVARS * (5 + 3) * 8
DEFAULT_SIZES = (16, 32, 48, 64)
DEFAULT_TILE = (32, 8)
TRAVERSALS = ("lex", "tiled")
BENCH_SEED = 20170907


def _shape3(n) -> tuple[int, int, int]:
    if np.isscalar(n):
        return (int(n),) * 3
    nx, ny, nz = (int(v) for v in n)
    return (nx, ny, nz)


def make_bench_values(shape, seed: int = BENCH_SEED) -> np.ndarray:
    """Canonical per-point values in [0.5, 1.5), shape (padded points, NVARS) (bench.py:45-50)."""
    nx, ny, nz = _shape3(shape)
    npts = (nx + 2 * X_PAD) * ny * nz
    rng = np.random.default_rng(seed)
    return 0.5 + rng.random((npts, NVARS))


def pack_values(values: np.ndarray, layout: Layout) -> np.ndarray:
    """One flat buffer per layout (bench.py:53-57)."""
    if layout == Layout.INTERLEAVED:
        return np.ascontiguousarray(values).reshape(-1)
    return np.ascontiguousarray(values.T).reshape(-1)


@dataclass
class BenchRecord:
    """One benchmarked configuration with its timing statistics (bench.py:60-99)."""

    shape: tuple[int, int, int]
    layout: Layout
    traversal: str
    times: list[float] = field(default_factory=list)
    wasted_lanes: int = 0

    @property
    def active_points(self) -> int:
        return self.shape[0] * self.shape[1] * self.shape[2]

    @property
    def median_seconds(self) -> float:
        return statistics.median(self.times)

    @property
    def min_seconds(self) -> float:
        return min(self.times)

    @property
    def cv(self) -> float:
        mean = statistics.fmean(self.times)
        return statistics.pstdev(self.times) / mean if mean > 0.0 else 0.0

    @property
    def bandwidth_gbs(self) -> float:
        return self.active_points * BYTES_PER_POINT / self.median_seconds / 1e9

    @property
    def wasted_fraction(self) -> float:
        visited = self.active_points + self.wasted_lanes
        return self.wasted_lanes / visited if visited else 0.0

    @property
    def size_label(self) -> str:
        nx, ny, nz = self.shape
        return str(nx) if nx == ny == nz else f"{nx}x{ny}x{nz}"


def run_case(shape, layout: Layout, traversal: str = "lex", repeats: int = 5,
             tile: tuple[int, int] = DEFAULT_TILE, params: WenoParams = DEFAULT_PARAMS,
             seed: int = BENCH_SEED) -> tuple[BenchRecord, np.ndarray]:
    """Time one (shape, layout, traversal) case on the current CUDA device;
    returns the record and the point-major weight output (bench.py:102-140)."""
    if traversal not in TRAVERSALS:
        raise ValueError(f"traversal must be one of {TRAVERSALS}, got {traversal!r}")
    if repeats < 1:
        raise ValueError("repeats must be at least 1")
    L = _lib.load(require_cuda=True)
    nx, ny, nz = _shape3(shape)
    data = torch.from_numpy(pack_values(make_bench_values((nx, ny, nz), seed), layout)).cuda()
    npts = (nx + 2 * X_PAD) * ny * nz
    out = torch.zeros(3 * NVARS * npts, dtype=torch.float64, device="cuda")
    record = BenchRecord(shape=(nx, ny, nz), layout=Layout(layout), traversal=traversal)
    stream = torch.cuda.current_stream()
    wasted = ctypes.c_int64(0)

    def run_once() -> None:
        _lib.check(L.hd_bench_weights(data.data_ptr(), int(layout), TRAVERSALS.index(traversal), nx, ny,
                                      nz, X_PAD, int(tile[0]), int(tile[1]), float(params.epsilon),
                                      int(params.power), out.data_ptr(), ctypes.byref(wasted),
                                      ctypes.c_void_p(stream.cuda_stream)), "hd_bench_weights")

    run_once()  # warm-up
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(repeats):
        torch.cuda.synchronize()
        e0.record(stream)
        run_once()
        e1.record(stream)
        e1.synchronize()
        record.times.append(e0.elapsed_time(e1) / 1e3)
    record.wasted_lanes = int(wasted.value)
    return record, out.cpu().numpy()


def layout_sweep(sizes=DEFAULT_SIZES, repeats: int = 5, traversals=("lex",),
                 tile: tuple[int, int] = DEFAULT_TILE) -> list[BenchRecord]:
    """Every size x layout x traversal combination (bench.py:143-156)."""
    records = []
    for n in sizes:
        for layout in (Layout.INTERLEAVED, Layout.COMPONENT_CONTIGUOUS):
            for traversal in traversals:
                rec, _ = run_case(n, layout, traversal, repeats=repeats, tile=tile)
                records.append(rec)
    return records


def _layout_name(layout: Layout) -> str:
    return "interleaved" if layout == Layout.INTERLEAVED else "contiguous"


def bench_report(records: list[BenchRecord]) -> str:
    """Text table ``n layout traversal median_s bandwidth_GBs ratio_vs_baseline``;
    the baseline of each size is its interleaved/lex row, else its first row
    (bench.py:163-189)."""
    baselines = {}
    for rec in records:
        key = rec.size_label
        if key not in baselines or (rec.layout == Layout.INTERLEAVED and rec.traversal == "lex"):
            baselines[key] = rec
    lines = ["n layout traversal median_s bandwidth_GBs ratio_vs_baseline"]
    for rec in records:
        ratio = rec.median_seconds / baselines[rec.size_label].median_seconds
        lines.append(f"{rec.size_label} {_layout_name(rec.layout)} {rec.traversal} "
                     f"{rec.median_seconds:.3g} {rec.bandwidth_gbs:.3g} {ratio:.3g}")
    if records:
        lines.append(f"# max_cv {max(rec.cv for rec in records):.3g}")
    return "\n".join(lines) + "\n"


def soft_ordering_checks(records: list[BenchRecord]) -> list[str]:
    """Expected-but-not-guaranteed orderings, reported as warnings (bench.py:192-221)."""
    notes = []
    by_key = {(r.size_label, r.layout, r.traversal): r for r in records}
    for size in sorted({r.size_label for r in records}):
        aos = by_key.get((size, Layout.INTERLEAVED, "lex"))
        soa = by_key.get((size, Layout.COMPONENT_CONTIGUOUS, "lex"))
        if aos and soa and soa.median_seconds > aos.median_seconds:
            notes.append(f"n={size}: contiguous layout was slower than interleaved "
                         f"({soa.median_seconds:.3g}s vs {aos.median_seconds:.3g}s)")
        for layout in (Layout.INTERLEAVED, Layout.COMPONENT_CONTIGUOUS):
            lex = by_key.get((size, layout, "lex"))
            tiled = by_key.get((size, layout, "tiled"))
            if lex and tiled and tiled.wasted_lanes > 0 and tiled.median_seconds < lex.median_seconds:
                notes.append(f"n={size} {_layout_name(layout)}: tiled traversal beat lexicographic "
                             f"despite wasting {tiled.wasted_fraction:.1%} of its lanes")
    for note in notes:
        warnings.warn(note, RuntimeWarning, stacklevel=2)
    return notes
