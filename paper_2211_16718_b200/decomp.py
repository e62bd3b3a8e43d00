"""Domain decomposition over GPUs: one process per GPU, NCCL halo exchange.

Mirrors pkg/src/hitdns/decomp.py (RankLayout, rank_of, coords_of,
decompose, default_dims, scatter, gather, parallel_advance, TimingReport,
comm_fraction) with the reference's thread ranks + queues (decomp.py:146-268)
replaced by torch.distributed over NCCL/NVLink:

* any 3D block decomposition of the reference (decomp.py:66-103); the
  default splits z only (dims = (1, 1, P)): z faces are contiguous planes per
  variable, so the halo is sent straight out of the state buffer with no pack
  kernel, and the x sweep never reads them; x and y faces of
  split axes are packed into contiguous buffers;
* the state face exchange of each RK stage is issued as one NCCL group
  (``batch_isend_irecv``) right after the previous stage's update kernel and
  overlaps the x sweep when x is not split (``hd_stage_part`` HD_PART_LOCAL /
  HD_PART_HALO);
* the viscous flux fields are exchanged along the axes that differentiate
  them; the z group (4 of the 9 symmetric flux fields, g planes) while the y
  sweep runs, before the z sweep that differentiates them;
* the CFL signal and diagnostics are combined with ``all_reduce`` (MAX for
  signals, SUM for totals) on device tensors -- dt never leaves HBM.

Because every kernel computes each point from the same inputs in the same
order, and MAX reductions are exact, a decomposed run reproduces the
single-GPU run bit-for-bit (the reference's invariant, test_decomp.py:194-204).
"""

from __future__ import annotations

import ctypes
import hashlib
import os
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


def _legal(dims, n, ghost_width: int) -> bool:
    return all(n[d] % dims[d] == 0 and n[d] // dims[d] >= ghost_width for d in range(3))


def default_dims(nranks: int, n, ghost_width: int = 3):
    """The reference's rank grid (decomp.py:106-140): among the legal factorings
    dx * dy * dz = nranks, the one with the least exchanged face area, ties to
    the larger x split, then the larger y split."""
    nranks = int(nranks)
    candidates = []
    for dx in (d for d in range(1, nranks + 1) if nranks % d == 0):
        for dy in (d for d in range(1, nranks // dx + 1) if (nranks // dx) % d == 0):
            dims = (dx, dy, nranks // (dx * dy))
            if not _legal(dims, n, ghost_width):
                continue
            loc = [n[d] // dims[d] for d in range(3)]
            area = sum(2 * loc[(d + 1) % 3] * loc[(d + 2) % 3] for d in range(3) if dims[d] > 1)
            candidates.append(((area, -dx, -dy), dims))
    if not candidates:
        raise ConfigError(f"no legal decomposition of {tuple(n)} into {nranks} ranks")
    return min(candidates)[1]


def gpu_dims(nranks: int, n, ghost_width: int = 3):
    """The GPU default of the drivers: z slabs (1, 1, nranks) when legal -- z faces
    are contiguous per variable (no pack kernels), the x/y sweeps overlap the
    exchange, and the peer-store halo needs no strided stores -- else the
    reference's choice (default_dims).  Results are decomposition-invariant,
    so this is purely a performance choice."""
    dims = (1, 1, int(nranks))
    return dims if _legal(dims, n, ghost_width) else default_dims(nranks, n, ghost_width)


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


class _Pending:
    """In-flight halo exchange: NCCL/gloo work handles plus the ghost slices
    that receive the packed x/y faces once the work completes."""

    def __init__(self, works=(), unpack=()):
        self.works = list(works)
        self.unpack = list(unpack)

    def wait(self) -> None:
        for w in self.works:
            w.wait()
        for dst, src in self.unpack:
            dst.copy_(src)
        self.works, self.unpack = [], []


class _WaitClock:
    """Exposed communication time of one rank (the reference's comm timer,
    decomp.py:202-221 and :359-361): each wait is bracketed by CUDA events on
    the compute stream, so what is measured is how long that stream stood still
    for a halo or a collective -- zero when the exchange finished behind the
    kernels it overlapped.  Host clock for CPU (gloo) tensors.  ``total()``
    synchronises once and drains the pairs."""

    def __init__(self):
        self.pairs = []
        self.host = 0.0

    def __call__(self, fn, cuda: bool = True):
        if not (cuda and torch.cuda.is_available() and torch.cuda.is_initialized()):
            t0 = _time.perf_counter()
            out = fn()
            self.host += _time.perf_counter() - t0
            return out
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = fn()
        b.record()
        self.pairs.append((a, b))
        return out

    def total(self) -> float:
        sec = self.host
        if self.pairs:
            self.pairs[-1][1].synchronize()
            sec += sum(a.elapsed_time(b) for a, b in self.pairs) / 1e3
        self.pairs, self.host = [], 0.0
        return sec


class DistHalo:
    """Ghost synchronisation of one rank over torch.distributed.

    Drop-in for the reference's RankHalo (decomp.py:183-241): ``sync_fields``
    and ``sync_scalars`` have the same meaning (axes in x, y, z order, each
    over the full ghosted extent of the others, so edges and corners match the
    monolithic fill); ``exchange_async`` is the overlapped form used by the
    fused march.  Any 3D block decomposition: an axis with one block wraps
    locally (periodic), a split axis exchanges g planes with its two
    neighbours.  z faces are contiguous per variable and are sent straight out
    of the buffer; x and y faces are packed into contiguous buffers (one copy
    kernel per face).  Works on CUDA tensors with NCCL and on CPU tensors with
    gloo (tests)."""

    def __init__(self, layout: RankLayout, group=None):
        self.layout = layout
        self.group = group
        self.periodic = tuple(layout.dims[d] == 1 for d in range(3))
        self.split = tuple(d for d in range(3) if layout.dims[d] > 1)
        self.comm_seconds = 0.0  # exposed halo/collective waits (_WaitClock), seconds
        self.clock = _WaitClock()
        self.lo = tuple(layout.neighbor(d, -1) for d in range(3))
        self.hi = tuple(layout.neighbor(d, +1) for d in range(3))

    def _peer(self, r: int) -> int:
        return r if self.group is None else dist.get_global_rank(self.group, r)

    def _axis_ops(self, v: torch.Tensor, fields, d: int, ops: list, unpack: list) -> None:
        """P2P ops moving g planes of each listed field of ``v`` (nf, gz, gy, gx)
        along axis d: my top interior planes to the high neighbour's low ghosts,
        my bottom interior planes to the low neighbour's high ghosts.  Issue
        order per field (send-hi, send-lo / recv-lo, recv-hi) matches pairwise
        FIFO order even when lo == hi (2 blocks along d)."""
        g = self.layout.spec.ghost_width
        n = v.shape[3 - d] - 2 * g
        dim = 3 - d  # tensor dim of axis d (fields, z, y, x)
        hi, lo = self._peer(self.hi[d]), self._peer(self.lo[d])
        for f in fields:
            fv = v[f]
            top, bot = fv.narrow(dim - 1, n, g), fv.narrow(dim - 1, g, g)
            lo_ghost, hi_ghost = fv.narrow(dim - 1, 0, g), fv.narrow(dim - 1, n + g, g)
            if d == 2:  # contiguous planes: no staging
                ops.append(dist.P2POp(dist.isend, top, hi, self.group))
                ops.append(dist.P2POp(dist.isend, bot, lo, self.group))
                ops.append(dist.P2POp(dist.irecv, lo_ghost, lo, self.group))
                ops.append(dist.P2POp(dist.irecv, hi_ghost, hi, self.group))
            else:
                r_lo, r_hi = torch.empty_like(lo_ghost, memory_format=torch.contiguous_format), \
                    torch.empty_like(hi_ghost, memory_format=torch.contiguous_format)
                ops.append(dist.P2POp(dist.isend, top.contiguous(), hi, self.group))
                ops.append(dist.P2POp(dist.isend, bot.contiguous(), lo, self.group))
                ops.append(dist.P2POp(dist.irecv, r_lo, lo, self.group))
                ops.append(dist.P2POp(dist.irecv, r_hi, hi, self.group))
                unpack += [(lo_ghost, r_lo), (hi_ghost, r_hi)]

    def exchange_async(self, buf: torch.Tensor, nfields: int, spec: GridSpec, axes=None,
                       fields=None) -> _Pending:
        """Exchange the split ``axes`` (default: all split axes) of fields
        ``fields`` (default: all ``nfields``) of the flat buffer ``buf`` as one
        NCCL group.  Faces of different axes go concurrently: the stencils are
        axis-aligned, so no edge or corner ghost is ever read."""
        axes = self.split if axes is None else tuple(d for d in axes if self.layout.dims[d] > 1)
        if not axes:
            return _Pending()
        v = buf[: nfields * spec.total_points].view((nfields,) + spec.shape)
        fields = range(nfields) if fields is None else fields
        ops, unpack = [], []
        for d in axes:
            self._axis_ops(v, fields, d, ops, unpack)
        return _Pending(dist.batch_isend_irecv(ops), unpack)

    def exchange_z_async(self, buf: torch.Tensor, nfields: int, spec: GridSpec) -> _Pending:
        return self.exchange_async(buf, nfields, spec, axes=(2,))

    @staticmethod
    def wait(pending) -> None:
        if isinstance(pending, _Pending):
            pending.wait()
        else:
            for w in pending:
                w.wait()

    @staticmethod
    def _wrap(buf: torch.Tensor, nfields: int, spec: GridSpec, d: int) -> None:
        """Local periodic wrap along axis d (grid.py:211-222), any device."""
        g = spec.ghost_width
        n = spec.n[d]
        v = buf.view((nfields,) + spec.shape)
        dim = 3 - d
        v.narrow(dim, 0, g).copy_(v.narrow(dim, n, g))
        v.narrow(dim, n + g, g).copy_(v.narrow(dim, g, g))

    def _sync(self, flat: torch.Tensor, nfields: int, spec: GridSpec) -> None:
        for d in range(3):
            if self.layout.dims[d] == 1:
                self._wrap(flat, nfields, spec, d)
            else:
                self.exchange_async(flat, nfields, spec, axes=(d,)).wait()

    def sync_fields(self, fields: FieldSet) -> FieldSet:
        """x, y, z in turn over full extents (decomp.py:223-234), so edges and
        corners match the monolithic fill."""
        t0 = _time.perf_counter()
        self._sync(fields.data, NVARS, fields.spec)
        self.comm_seconds += _time.perf_counter() - t0
        return fields

    def sync_scalars(self, arrays, n, g: int) -> None:
        spec = GridSpec(tuple(n), ghost_width=g)
        for arr in arrays:
            self._sync(arr.reshape(-1), 1, spec)

    def sync_flux_fields(self, vflux: torch.Tensor, spec: GridSpec) -> None:
        """The viscous flux groups' faces along the axes that differentiate them
        (the sync_scalars of viscous.py:118 for a decomposed parabolic_rhs)."""
        for d in self.split:
            self.exchange_async(vflux, 9, spec, axes=(d,), fields=_VF_GROUP[d]).wait()

    # ---- fused march --------------------------------------------------------
    def advance(self, fields: FieldSet, gas: GasModel, tparams, weno_params: WenoParams,
                delta: float, t0: float, observer, dt_provider, mode):
        """The decomposed RK march.  Per stage (hd_stage_part):

        * state faces of the stage input go out as one group; the LOCAL x sweep
          overlaps them unless x itself is split (exact mode's LOCAL part also
          sweeps y, so it waits for a y split too);
        * HALO (viscous fluxes) needs every state ghost;
        * the viscous flux groups are exchanged along their own axes: the x and
          y groups before MID (y sweep + D_x F_x + D_y F_y), the z group while
          MID runs, before UPDATE (z sweep + D_z F_z + RK update)."""
        from .plan import get_plan
        from .timeint import _SCHEME_CODE, _as_device, _DeviceMarch

        fields = _as_device(fields)  # host (pinned) buffers are uploaded once
        spec = fields.spec
        plan = get_plan(spec, gas, weno_params, delta, mode, periodic=self.periodic)
        if self.peer_enabled(fields) and _PeerLink.get(self).attach(plan):
            return self._advance_peer(plan, fields, gas, tparams, t0, observer, dt_provider)
        exact = plan.mode == "exact"
        scheme = _SCHEME_CODE[tparams.scheme]
        nst = 3 if scheme == _lib.HD_SCHEME_RK3 else 4
        vflux = plan.fields(_lib.HD_BUF_VFLUX, 9)
        visc = gas.effective_mu != 0.0
        halo = self
        local_waits = 0 in self.split or (exact and 1 in self.split)
        pre_mid = tuple(d for d in (0, 1) if d in self.split)

        clock = self.clock

        def stepper(u, dt_dev, tag):
            plan.fill_ghosts(u, NVARS)  # periodic axes wrap locally; split axes exchanged below
            for s in range(nst):
                us = plan.stage_input(scheme, s, u)
                pend = halo.exchange_async(us, NVARS, spec)
                if local_waits:
                    clock(pend.wait)
                plan.stage_part(scheme, s, _lib.HD_PART_LOCAL, u, dt_dev, tag)
                clock(pend.wait)
                plan.stage_part(scheme, s, _lib.HD_PART_HALO, u, dt_dev, tag)
                if visc and pre_mid:
                    for d in pre_mid:
                        clock(halo.exchange_async(vflux, 9, spec, axes=(d,), fields=_VF_GROUP[d]).wait)
                zpend = (halo.exchange_async(vflux, 9, spec, axes=(2,), fields=_VF_GROUP[2])
                         if visc else _Pending())
                plan.stage_part(scheme, s, _lib.HD_PART_MID, u, dt_dev, tag)  # overlaps it
                clock(zpend.wait)
                plan.stage_part(scheme, s, _lib.HD_PART_UPDATE, u, dt_dev, tag)

        def reducer(red):
            if self.split:
                clock(lambda: _combine_reductions(red, halo.group))

        def ghost_sync(u):
            plan.fill_ghosts(u, NVARS)
            clock(halo.exchange_async(u, NVARS, spec).wait)

        nblocks = self.layout.dims[0] * self.layout.dims[1] * self.layout.dims[2]
        march = _DeviceMarch(plan, fields, gas, tparams, t0, stepper=stepper, reducer=reducer,
                             global_points=spec.interior_points * nblocks,
                             error_combine=lambda key: _combine_error_key(key, self.group),
                             ghost_sync=ghost_sync,
                             sum_combine=lambda t: _combine_sums(t, self.group))
        try:
            return march.run(observer, dt_provider)
        finally:
            self.comm_seconds += clock.total()

    def peer_enabled(self, fields: FieldSet) -> bool:
        """Blocks on CUDA: the halo goes over NVLink peer stores (hd_peer_*)
        instead of NCCL, unless HD_PEER=0."""
        return (bool(self.split) and fields.data.is_cuda
                and os.environ.get("HD_PEER", "1") not in ("0", ""))

    def _advance_peer(self, plan, fields: FieldSet, gas: GasModel, tparams, t0, observer,
                      dt_provider):
        """The block march with the halo fused into the producing kernels: the z
        sweep's RK update and the flux kernel store their boundary layers into
        the neighbours' ghost layers over NVLink along every split axis; per RK
        stage v (fast mode, z split only)

            LOCAL; wait(state >= v-1); HALO; signal(vflux, v); MID;
            wait(vflux >= v); UPDATE; signal(state, v)

        with the state wait moved before LOCAL when x is split (the x sweep reads
        x ghosts) and the flux wait before MID when x or y is split (the y sweep
        differentiates the x and y flux groups) (include/hd.h, hd_peer.cu).  The
        march state lives in the plan's HD_BUF_STATE so the peers' images land at
        the same offsets."""
        from .timeint import _SCHEME_CODE, _DeviceMarch

        spec = fields.spec
        scheme = _SCHEME_CODE[tparams.scheme]
        nst = 3 if scheme == _lib.HD_SCHEME_RK3 else 4
        visc = gas.effective_mu != 0.0
        state = plan.fields(_lib.HD_BUF_STATE, NVARS)
        state.copy_(fields.data)
        local = FieldSet(spec, Layout.COMPONENT_CONTIGUOUS, state)
        try:
            self._sync(state, NVARS, spec)  # initial ghosts (wrap + NCCL faces, once)
            counter = [0]

            # LOCAL reads x ghosts (exact mode: also y); MID reads the x/y flux groups
            exact = plan.mode == "exact"
            state_before_local = 0 in self.split or (exact and 1 in self.split)
            vflux_before_mid = not exact and (0 in self.split or 1 in self.split)

            clock = self.clock

            def wait(which, v):  # the spin kernel's duration = the exposed wait
                clock(lambda: plan.peer_wait(which, v))

            def stepper(u, dt_dev, tag):
                plan.fill_ghosts(u, NVARS)  # periodic axes wrap; split axes arrive as peer stores
                for s in range(nst):
                    v = counter[0] + 1
                    if state_before_local:
                        wait(_lib.HD_PEER_STATE, v - 1)
                    plan.stage_part(scheme, s, _lib.HD_PART_LOCAL, u, dt_dev, tag)
                    if not state_before_local:
                        wait(_lib.HD_PEER_STATE, v - 1)
                    plan.stage_part(scheme, s, _lib.HD_PART_HALO, u, dt_dev, tag)
                    if visc:
                        plan.peer_signal(_lib.HD_PEER_VFLUX, v)
                        if vflux_before_mid:
                            wait(_lib.HD_PEER_VFLUX, v)
                    plan.stage_part(scheme, s, _lib.HD_PART_MID, u, dt_dev, tag)
                    if visc and not vflux_before_mid:
                        wait(_lib.HD_PEER_VFLUX, v)
                    plan.stage_part(scheme, s, _lib.HD_PART_UPDATE, u, dt_dev, tag)
                    plan.peer_signal(_lib.HD_PEER_STATE, v)
                    counter[0] = v

            def reducer(red):
                clock(lambda: _combine_reductions(red, self.group))

            def ghost_sync(u):
                # the last UPDATE stored this rank's boundary layers into the
                # neighbours' ghosts (and theirs into ours) and signalled
                wait(_lib.HD_PEER_STATE, counter[0])
                plan.fill_ghosts(u, NVARS)

            def protocol_check():
                # a wait that timed out on any rank ends the march on every rank, at the
                # next check (every step when the march synchronises, else at its end)
                flag = torch.tensor([1 if plan.peer_timed_out() else 0], dtype=torch.int64,
                                    device=state.device)
                dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=self.group)
                _check_protocol(not bool(flag.item()), "a neighbour never signalled (peer halo timed out)")

            nblocks = self.layout.dims[0] * self.layout.dims[1] * self.layout.dims[2]
            march = _DeviceMarch(plan, local, gas, tparams, t0, stepper=stepper, reducer=reducer,
                                 global_points=spec.interior_points * nblocks,
                                 copy=False,
                                 error_combine=lambda key: _combine_error_key(key, self.group),
                                 ghost_sync=ghost_sync,
                                 sum_combine=lambda t: _combine_sums(t, self.group),
                                 protocol_check=protocol_check)
            try:
                res = march.run(observer, dt_provider)
            finally:
                self.comm_seconds += clock.total()
            flag = torch.tensor([1 if plan.peer_timed_out() else 0], dtype=torch.int64,
                                device=state.device)
            dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=self.group)
            timed_out = bool(flag.item())
        finally:
            plan.peer_attach([None] * 3, [None] * 3)  # the mapping stays cached (_PeerLink)
        _check_protocol(not timed_out, "a z neighbour never signalled (peer halo timed out)")
        res.fields = FieldSet(spec, Layout.COMPONENT_CONTIGUOUS, state.clone())
        return res


def _combine_reductions(red: torch.Tensor, group) -> None:
    """The per-step reduction over ranks in one collective: all-gather the
    HD_RED_* vectors, then MAX the signals (exact) and SUM the totals in rank
    order (deterministic) on the device."""
    world = dist.get_world_size(group)
    allv = torch.empty((world, red.numel()), dtype=red.dtype, device=red.device)
    dist.all_gather_into_tensor(allv, red.contiguous(), group=group)
    red[0:3] = allv[:, 0:3].amax(dim=0)
    acc = allv[0, 3:].clone()
    for r in range(1, world):
        acc += allv[r, 3:]
    red[3:] = acc


def _combine_sums(t: torch.Tensor, group) -> None:
    """In place: the sum over ranks, added in rank order (deterministic)."""
    world = dist.get_world_size(group)
    allv = torch.empty((world, t.numel()), dtype=t.dtype, device=t.device)
    dist.all_gather_into_tensor(allv, t.contiguous().view(-1), group=group)
    acc = allv[0].clone()
    for r in range(1, world):
        acc += allv[r]
    t.view(-1).copy_(acc)


def _combine_error_key(key: int, group) -> int:
    """Earliest error over all ranks (0 = none): the key orders by step, stage,
    code, then point, so MIN picks the error every rank must raise."""
    none = (1 << 63) - 1
    t = torch.tensor([key if key else none], dtype=torch.int64,
                     device=torch.device("cuda", torch.cuda.current_device())
                     if dist.get_backend(group) == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    v = int(t.item())
    return 0 if v == none else v


class _PeerLink:
    """The z neighbours' plan workspaces mapped into this process (CUDA IPC).

    Mappings are kept across marches (opening an IPC handle costs milliseconds):
    each march all-gathers a 64-bit digest of every rank's (handle, offset) and
    re-opens only what changed (a neighbour's plan was rebuilt)."""

    _cache: dict = {}

    def __init__(self, halo: "DistHalo"):
        self.halo = halo
        self.L = _lib.load()
        self.digests = None
        self.handles = None
        self.opened = {}  # group rank -> (mapped pointer, offset)

    @classmethod
    def get(cls, halo: "DistHalo") -> "_PeerLink":
        key = (id(halo.group), halo.layout.rank, halo.layout.dims)
        link = cls._cache.get(key)
        if link is None:
            link = cls._cache[key] = cls(halo)
        link.halo = halo
        return link

    def attach(self, plan) -> bool:
        """Map/attach the neighbours; False on every rank if any rank cannot."""
        halo = self.halo
        world = dist.get_world_size(halo.group)
        handle, off = plan.ipc_handle()
        digest = int.from_bytes(hashlib.blake2b(handle + off.to_bytes(8, "little"),
                                                digest_size=8).digest(), "little", signed=True)
        dev = torch.device("cuda", torch.cuda.current_device())
        mine = torch.tensor([digest], dtype=torch.int64, device=dev)
        alld = [torch.empty_like(mine) for _ in range(world)]
        torch.cuda.synchronize()
        dist.all_gather(alld, mine, group=halo.group)  # also: every rank finished its last march
        digests = [int(t.item()) for t in alld]
        if digests != self.digests:
            allh = [None] * world
            dist.all_gather_object(allh, (handle, off), group=halo.group)
            self.release()
            ok = 1
            for r in {n for d in halo.split for n in (halo.lo[d], halo.hi[d])}:
                h, o = allh[r]
                ptr = ctypes.c_void_p()
                if self.L.hd_ipc_open(ctypes.create_string_buffer(h, 64), o, ctypes.byref(ptr)) != 0:
                    ok = 0  # no IPC/P2P between these processes (e.g. no shared IPC namespace)
                    break
                self.opened[r] = (ptr.value, o)
            flag = torch.tensor([ok], dtype=torch.int64, device=dev)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=halo.group)
            if not int(flag.item()):
                self.release()
                return False  # every rank falls back to the NCCL halo together
            self.digests = digests
        lo = [self.opened[halo.lo[d]][0] if d in halo.split else None for d in range(3)]
        hi = [self.opened[halo.hi[d]][0] if d in halo.split else None for d in range(3)]
        plan.peer_attach(lo, hi)  # zeroes the flags
        torch.cuda.synchronize()
        dist.barrier(group=halo.group)  # every rank's flags are zero before anyone signals
        return True

    def release(self) -> None:
        for ptr, off in self.opened.values():
            self.L.hd_ipc_close(ctypes.c_void_p(ptr), off)
        self.opened = {}
        self.digests = None


# symmetric viscous flux fields (tau00 tau01 tau11 w0 w1 | tau02 tau12 tau22 w2) that
# the divergence differentiates along each axis (hd_device.cuh vf_field)
_VF_GROUP = ((0, 1, 5, 3), (1, 2, 6, 4), (5, 6, 7, 8))


def parallel_advance(fields: FieldSet, gas: GasModel, tparams, weno_params: WenoParams = DEFAULT_PARAMS,
                     delta: float = 0.0, dims=None, workers_per_rank: int = 1, group=None,
                     mode: str | None = None) -> ParallelResult:
    """Decomposed march; returns the gathered global state on every rank
    (decomp.py:328-407).  SPMD: every rank of ``group`` (default: the world)
    calls it with the same global ``fields``; one rank per GPU.  For the best
    overlap of the halo with the sweeps, initialise NCCL with
    ``TORCH_NCCL_HIGH_PRIORITY=1`` (bench.py and the CLI do)."""
    from .timeint import advance

    fields = fields if isinstance(fields, FieldSet) else FieldSet.from_numpy(fields)
    if fields.layout != Layout.COMPONENT_CONTIGUOUS:
        raise ValueError("parallel_advance needs COMPONENT_CONTIGUOUS fields")
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    if dims is None:
        dims = gpu_dims(world, fields.spec.n, fields.spec.ghost_width)
    dims = tuple(int(d) for d in dims)
    if dims[0] * dims[1] * dims[2] != world:
        raise ConfigError(f"dims {dims} need {dims[0] * dims[1] * dims[2]} ranks, have {world}")
    layouts = decompose(fields.spec, dims)
    lay = layouts[rank]
    local = scatter(fields, [lay])[0]
    wall0 = _time.perf_counter()
    comm = 0.0
    if world == 1:
        res = advance(local, gas, tparams, weno_params, delta, mode=mode)
    else:
        halo = DistHalo(lay, group)
        res = halo.advance(local, gas, tparams, weno_params, delta, 0.0, None, None, mode)
        comm = halo.comm_seconds
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
    # one report per rank, as the reference (decomp.py:380-391): comm = the rank's
    # exposed halo/collective waits, comp = the rest of its wall time
    mine = torch.tensor([wall, max(wall - comm, 0.0), comm], dtype=torch.float64,
                        device=fields.data.device if fields.data.is_cuda else "cpu")
    if world > 1:
        every = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(every, mine, group=group)
    else:
        every = [mine]
    reports = [TimingReport(r, dims, res.steps, *(float(x) for x in every[r].tolist()))
               for r in range(world)]
    return ParallelResult(fields=gathered, t=res.t, reports=reports)


def _check_protocol(ok: bool, what: str) -> None:
    if not ok:
        raise HaloProtocolError(what)


@dataclass
class ScaleRow:
    """decomp.py:414-423."""

    ranks: int
    dims: tuple
    wall_seconds: float
    comp_seconds: float
    comm_seconds: float

    @property
    def ratio(self) -> float:
        return comm_fraction(self.comm_seconds, self.comm_seconds + self.comp_seconds)


def strong_scaling(fields: FieldSet, gas: GasModel, tparams, ranks_list,
                   weno_params: WenoParams = DEFAULT_PARAMS, delta: float = 0.0, dims_for=None,
                   mode: str | None = None) -> list:
    """The same run over rank counts from identical initial fields
    (decomp.py:426-461), one process per GPU: every rank of the world calls
    it; a rank count outside 1..world size raises ConfigError (one process per
    GPU: the reference's thread ranks have no such limit).  Each count runs on a
    sub-group of the first ``nranks`` ranks (the others wait at a barrier)
    after a one-step warm-up on that group; ``wall`` is the slowest rank's
    device-synchronised wall clock.  Rank 0 gets the rows; the others get []."""
    from .timeint import TimeParams

    world = dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank() if world > 1 else 0
    warm = TimeParams(scheme=tparams.scheme, dt=tparams.dt, cfl=tparams.cfl,
                      cfl_mode=tparams.cfl_mode, max_steps=1)
    counts = [int(r) for r in ranks_list]
    bad = [r for r in counts if r < 1 or r > world]
    if bad:
        raise ConfigError(f"rank counts {bad} cannot run on {world} process(es) "
                          f"(one per GPU; launch with --nproc-per-node >= {max(counts)})")
    rows = []
    for nranks in counts:
        dims = dims_for(nranks) if dims_for else gpu_dims(nranks, fields.spec.n, fields.spec.ghost_width)
        group = None
        if world > 1:
            group = dist.new_group(list(range(nranks)))
        row = [0.0, 0.0, 0.0]
        if rank < nranks:
            sub = group if world > 1 else None
            parallel_advance(fields.copy(), gas, warm, weno_params, delta, dims, group=sub, mode=mode)
            res = parallel_advance(fields.copy(), gas, tparams, weno_params, delta, dims, group=sub,
                                   mode=mode)
            # decomp.py:452-460: slowest rank's wall; comp and comm summed over ranks
            row = [max(r.wall_seconds for r in res.reports), sum(r.comp_seconds for r in res.reports),
                   sum(r.comm_seconds for r in res.reports)]
        if world > 1:
            dev = fields.data.device if fields.data.is_cuda else torch.device("cpu")
            t = torch.tensor(row, dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)  # rank 0 of the sub-group holds the row
            row = t.tolist()
        rows.append(ScaleRow(nranks, tuple(dims), *row))
    return rows if rank == 0 else []


def scaling_report(rows) -> str:
    """``ranks dims wall comp comm ratio speedup efficiency`` (decomp.py:464-476)."""
    lines = ["ranks dims wall comp comm ratio speedup efficiency"]
    base = rows[0].wall_seconds if rows else 0.0
    for row in rows:
        speedup = base / row.wall_seconds if row.wall_seconds > 0.0 else 0.0
        lines.append(f"{row.ranks} {'x'.join(str(d) for d in row.dims)} {row.wall_seconds:.6f} "
                     f"{row.comp_seconds:.6f} {row.comm_seconds:.6f} {row.ratio:.4f} {speedup:.3f} "
                     f"{speedup / row.ranks:.3f}")
    return "\n".join(lines) + "\n"
