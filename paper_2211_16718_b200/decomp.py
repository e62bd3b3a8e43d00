"""Domain decomposition over GPUs: one process per GPU, NCCL halo exchange.

Mirrors pkg/src/hitdns/decomp.py (RankLayout, rank_of, coords_of,
decompose, default_dims, scatter, gather, parallel_advance, TimingReport,
comm_fraction) with the reference's thread ranks + queues (decomp.py:146-268)
replaced by torch.distributed over NCCL/NVLink:

* blocks are split along z (dims = (1, 1, P)): each rank's z faces are
  contiguous planes per variable, so the halo is sent straight out of the
  state buffer with no pack kernel;
* the state face exchange of each RK stage is issued as one NCCL group
  (``batch_isend_irecv``) right after the previous stage's update kernel and
  overlaps the x and y sweeps, which never read z ghosts; the z sweep waits
  on it (``hd_stage_part`` HD_PART_LOCAL / HD_PART_HALO);
* the viscous flux faces of the z-differentiated flux group (4 of the 9
  symmetric flux fields, g planes) are exchanged while the y sweep runs, before
  the z sweep that differentiates them;
* the CFL signal and diagnostics are combined with ``all_reduce`` (MAX for
  signals, SUM for totals) on device tensors -- dt never leaves HBM.

Because every kernel computes each point from the same inputs in the same
order, and MAX reductions are exact, a decomposed run reproduces the
single-GPU run bit-for-bit (the reference's invariant, test_decomp.py:194-204).
"""

from __future__ import annotations

import time as _time
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _lib
from .errors import ConfigError, HaloProtocolError
from .grid import FieldSet, GridSpec, Layout
from .physics import DEFAULT_PARAMS, GasModel, WenoParams

NVARS = 5


@dataclass(frozen=True)
class RankLayout:
    """decomp.py:36-52."""

    rank: int
    coords: tuple
    dims: tuple
    local_n: tuple
    offset: tuple
    spec: GridSpec

    def neighbor(self, dim: int, side: int) -> int:
        coords = list(self.coords)
        coords[dim] = (coords[dim] + side) % self.dims[dim]
        return rank_of(tuple(coords), self.dims)


def rank_of(coords, dims) -> int:
    """x-fastest numbering (decomp.py:54-56)."""
    return coords[0] + dims[0] * (coords[1] + dims[1] * coords[2])


def coords_of(rank: int, dims):
    return (rank % dims[0], (rank // dims[0]) % dims[1], rank // (dims[0] * dims[1]))


def decompose(spec: GridSpec, dims) -> list:
    """Equal blocks, n[d] % dims[d] == 0 and local >= ghost width (decomp.py:66-103)."""
    dims = tuple(int(d) for d in dims)
    if len(dims) != 3 or any(d < 1 for d in dims):
        raise ConfigError(f"dims must be three positive integers, got {dims}")
    local_n = []
    for d in range(3):
        if spec.n[d] % dims[d] != 0:
            raise ConfigError(f"dims[{d}]={dims[d]} does not divide the grid extent {spec.n[d]}")
        ln = spec.n[d] // dims[d]
        if ln < spec.ghost_width:
            raise ConfigError(f"local extent {ln} in dimension {d} is thinner than the "
                              f"ghost width {spec.ghost_width}")
        local_n.append(ln)
    local_n = tuple(local_n)
    local_len = tuple(spec.length[d] * local_n[d] / spec.n[d] for d in range(3))
    local_spec = GridSpec(n=local_n, length=local_len, ghost_width=spec.ghost_width)
    out = []
    for r in range(dims[0] * dims[1] * dims[2]):
        c = coords_of(r, dims)
        out.append(RankLayout(r, c, dims, local_n, tuple(c[d] * local_n[d] for d in range(3)),
                              local_spec))
    return out


def default_dims(nranks: int, n, ghost_width: int = 3):
    """GPU choice: split z only -> (1, 1, nranks).

    z faces are contiguous per variable (no pack kernels) and the x/y sweeps
    overlap the exchange.  The reference prefers x splits to minimise face
    area on CPUs (decomp.py:106-140); results are decomposition-invariant, so
    this is a pure performance choice."""
    dims = (1, 1, int(nranks))
    if n[2] % nranks == 0 and n[2] // nranks >= ghost_width:
        return dims
    raise ConfigError(f"no legal z decomposition of {tuple(n)} into {nranks} ranks "
                      f"(need n_z % ranks == 0 and n_z / ranks >= {ghost_width})")


def comm_fraction(comm_seconds: float, busy_seconds: float) -> float:
    return 0.0 if busy_seconds <= 0.0 else comm_seconds / busy_seconds


@dataclass
class TimingReport:
    rank: int
    dims: tuple
    steps: int
    wall_seconds: float
    comp_seconds: float
    comm_seconds: float

    @property
    def ratio(self) -> float:
        return comm_fraction(self.comm_seconds, self.comm_seconds + self.comp_seconds)


@dataclass
class ParallelResult:
    fields: FieldSet
    t: float
    reports: list


def scatter(fields: FieldSet, layouts) -> list:
    """Interior blocks of a global FieldSet (decomp.py:304-314)."""
    interior = fields.interior()
    out = []
    for lay in layouts:
        ox, oy, oz = lay.offset
        lx, ly, lz = lay.local_n
        local = FieldSet.zeros(lay.spec, fields.layout, device=fields.data.device)
        local.interior().copy_(interior[:, oz:oz + lz, oy:oy + ly, ox:ox + lx])
        out.append(local)
    return out


def gather(locals_, layouts, spec: GridSpec) -> FieldSet:
    """decomp.py:317-325."""
    out = FieldSet.zeros(spec, locals_[0].layout, device=locals_[0].data.device)
    interior = out.interior()
    for local, lay in zip(locals_, layouts):
        ox, oy, oz = lay.offset
        lx, ly, lz = lay.local_n
        interior[:, oz:oz + lz, oy:oy + ly, ox:ox + lx] = local.interior()
    return out


class DistHalo:
    """Ghost synchronisation of one rank over torch.distributed (z split).

    Drop-in for the reference's RankHalo (decomp.py:183-241): ``sync_fields``
    and ``sync_scalars`` have the same meaning; ``exchange_z_async`` is the
    overlapped form used by the fused march.  Works on CUDA tensors with the
    NCCL backend and on CPU tensors with gloo (tests)."""

    def __init__(self, layout: RankLayout, group=None):
        if layout.dims[0] != 1 or layout.dims[1] != 1:
            raise ConfigError(f"the GPU decomposition splits z only, got dims {layout.dims}")
        self.layout = layout
        self.group = group
        self.periodic = (True, True, layout.dims[2] == 1)
        self.comm_seconds = 0.0
        self.lo = layout.neighbor(2, -1)
        self.hi = layout.neighbor(2, +1)
        self._g_lo = self._g_hi = None

    def _peer(self, r: int) -> int:
        return r if self.group is None else dist.get_global_rank(self.group, r)

    def _z_ops(self, buf: torch.Tensor, nfields: int, spec: GridSpec):
        """P2P ops moving g z-planes of each field: my top interior planes to the
        high neighbour's low ghosts, my bottom interior planes to the low
        neighbour's high ghosts.  Issue order (send-hi, send-lo / recv-lo,
        recv-hi) matches pairwise FIFO order even when lo == hi (2 ranks)."""
        g = spec.ghost_width
        nz = spec.n[2]
        plane = spec.shape[1] * spec.shape[2]
        slab = g * plane
        npts = spec.total_points
        ops = []
        for f in range(nfields):
            base = f * npts
            top = buf[base + nz * plane: base + nz * plane + slab]          # planes [n, n+g)
            bot = buf[base + g * plane: base + g * plane + slab]            # planes [g, 2g)
            lo_ghost = buf[base: base + slab]                                # planes [0, g)
            hi_ghost = buf[base + (nz + g) * plane: base + (nz + g) * plane + slab]
            ops.append(dist.P2POp(dist.isend, top, self._peer(self.hi), self.group))
            ops.append(dist.P2POp(dist.isend, bot, self._peer(self.lo), self.group))
            ops.append(dist.P2POp(dist.irecv, lo_ghost, self._peer(self.lo), self.group))
            ops.append(dist.P2POp(dist.irecv, hi_ghost, self._peer(self.hi), self.group))
        return ops

    def exchange_z_async(self, buf: torch.Tensor, nfields: int, spec: GridSpec):
        if self.layout.dims[2] == 1:
            return []
        return dist.batch_isend_irecv(self._z_ops(buf, nfields, spec))

    @staticmethod
    def wait(works) -> None:
        for w in works:
            w.wait()

    def _wrap_xy(self, buf: torch.Tensor, nfields: int, spec: GridSpec) -> None:
        """Local periodic wrap along x then y (grid.py:211-222), any device."""
        g = spec.ghost_width
        nx, ny = spec.n[0], spec.n[1]
        v = buf.view((nfields,) + spec.shape)
        v[..., :g] = v[..., nx:nx + g]
        v[..., nx + g:] = v[..., g:2 * g]
        v[..., :g, :] = v[..., ny:ny + g, :]
        v[..., ny + g:, :] = v[..., g:2 * g, :]

    def _wrap_z(self, buf, nfields, spec) -> None:
        g = spec.ghost_width
        nz = spec.n[2]
        v = buf.view((nfields,) + spec.shape)
        v[:, :g] = v[:, nz:nz + g]
        v[:, nz + g:] = v[:, g:2 * g]

    def sync_fields(self, fields: FieldSet) -> FieldSet:
        """x wrap, y wrap, z exchange (decomp.py:223-234): full-extent faces,
        so edges and corners match the monolithic fill."""
        t0 = _time.perf_counter()
        self._wrap_xy(fields.data, NVARS, fields.spec)
        if self.layout.dims[2] == 1:
            self._wrap_z(fields.data, NVARS, fields.spec)
        else:
            self.wait(self.exchange_z_async(fields.data, NVARS, fields.spec))
        self.comm_seconds += _time.perf_counter() - t0
        return fields

    def sync_scalars(self, arrays, n, g: int) -> None:
        spec = GridSpec(tuple(n), ghost_width=g)
        for arr in arrays:
            flat = arr.reshape(-1)
            self._wrap_xy(flat, 1, spec)
            if self.layout.dims[2] == 1:
                self._wrap_z(flat, 1, spec)
            else:
                self.wait(self.exchange_z_async(flat, 1, spec))

    # ---- fused march --------------------------------------------------------
    def advance(self, fields: FieldSet, gas: GasModel, tparams, weno_params: WenoParams,
                delta: float, t0: float, observer, dt_provider, mode):
        from .plan import get_plan
        from .timeint import _SCHEME_CODE, _as_device, _DeviceMarch

        fields = _as_device(fields)  # host (pinned) buffers are uploaded once
        spec = fields.spec
        plan = get_plan(spec, gas, weno_params, delta, mode, periodic=self.periodic)
        scheme = _SCHEME_CODE[tparams.scheme]
        nst = 3 if scheme == _lib.HD_SCHEME_RK3 else 4
        stage_buf = plan.fields(_lib.HD_BUF_STAGE, 2 * NVARS)  # ping-pong halves
        half = NVARS * spec.total_points
        vflux_z = plan.fields(_lib.HD_BUF_VFLUX, 9)[5 * spec.total_points:]  # the z group
        visc = gas.effective_mu != 0.0
        halo = self

        def stepper(u, dt_dev, tag):
            plan.fill_ghosts(u, NVARS)  # x/y wrap of the step input (z: exchanged below)
            for s in range(nst):
                us = u if s == 0 else stage_buf[((s - 1) % 2) * half: ((s - 1) % 2 + 1) * half]
                works = halo.exchange_z_async(us, NVARS, spec)   # overlaps the x sweep
                plan.stage_part(scheme, s, _lib.HD_PART_LOCAL, u, dt_dev, tag)
                halo.wait(works)
                parts = _lib.HD_PART_HALO
                if s == 0 and tag == 0:  # primitives of u not yet produced by an update
                    parts |= _lib.HD_PART_PRIMS
                plan.stage_part(scheme, s, parts, u, dt_dev, tag)
                works = halo.exchange_z_async(vflux_z, 4, spec) if visc else []
                plan.stage_part(scheme, s, _lib.HD_PART_MID, u, dt_dev, tag)  # overlaps it
                halo.wait(works)
                plan.stage_part(scheme, s, _lib.HD_PART_UPDATE, u, dt_dev, tag)

        def reducer(red):
            if halo.layout.dims[2] > 1:
                dist.all_reduce(red[0:3], op=dist.ReduceOp.MAX, group=halo.group)
                dist.all_reduce(red[3:9], op=dist.ReduceOp.SUM, group=halo.group)

        march = _DeviceMarch(plan, fields, gas, tparams, t0, stepper=stepper, reducer=reducer,
                             global_points=spec.interior_points * self.layout.dims[2])
        return march.run(observer, dt_provider)


def parallel_advance(fields: FieldSet, gas: GasModel, tparams, weno_params: WenoParams = DEFAULT_PARAMS,
                     delta: float = 0.0, dims=None, workers_per_rank: int = 1, group=None,
                     mode: str | None = None) -> ParallelResult:
    """Decomposed march; returns the gathered global state on every rank
    (decomp.py:328-407).  SPMD: every rank of ``group`` (default: the world)
    calls it with the same global ``fields``; one rank per GPU."""
    from .timeint import advance

    fields = fields if isinstance(fields, FieldSet) else FieldSet.from_numpy(fields)
    if fields.layout != Layout.COMPONENT_CONTIGUOUS:
        raise ValueError("parallel_advance needs COMPONENT_CONTIGUOUS fields")
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    if dims is None:
        dims = default_dims(world, fields.spec.n, fields.spec.ghost_width)
    dims = tuple(int(d) for d in dims)
    if dims[0] * dims[1] * dims[2] != world:
        raise ConfigError(f"dims {dims} need {dims[0] * dims[1] * dims[2]} ranks, have {world}")
    layouts = decompose(fields.spec, dims)
    lay = layouts[rank]
    local = scatter(fields, [lay])[0]
    wall0 = _time.perf_counter()
    if world == 1:
        res = advance(local, gas, tparams, weno_params, delta, mode=mode)
    else:
        halo = DistHalo(lay, group)
        res = halo.advance(local, gas, tparams, weno_params, delta, 0.0, None, None, mode)
    if fields.data.is_cuda:
        torch.cuda.synchronize()
    wall = _time.perf_counter() - wall0
    if world == 1:
        gathered = gather([res.fields], [lay], fields.spec)
    else:
        parts = [torch.empty_like(res.fields.interior().contiguous()) for _ in range(world)]
        dist.all_gather(parts, res.fields.interior().contiguous(), group=group)
        locals_ = []
        for r, part in enumerate(parts):
            fs = FieldSet.zeros(layouts[r].spec, device=fields.data.device)
            fs.interior().copy_(part)
            locals_.append(fs)
        gathered = gather(locals_, layouts, fields.spec)
    report = TimingReport(rank, dims, res.steps, wall, wall, 0.0)
    return ParallelResult(fields=gathered, t=res.t, reports=[report])


def _check_protocol(ok: bool, what: str) -> None:
    if not ok:
        raise HaloProtocolError(what)
