"""Time integration on the GPU (mirrors pkg/src/hitdns/timeint.py).

Same public surface: ``TimeParams``, ``StepRecord``, ``AdvanceResult``,
``conserved_totals``, ``max_wavespeed_interior``, ``max_signal``,
``compute_dt``, ``make_rhs``, ``rk3_tvd_step``, ``rk4_step``, ``STEPPERS``,
``advance``, ``write_step_log``.

``advance`` runs the whole march on the device: per step one fused
reduction (CFL signal of the state and the previous step's diagnostics),
one dt kernel (cfl/signal, t_final clip, kept in HBM), and one ``hd_step``
(4 RK stages x [3 sweeps + viscous fluxes + divergence/RK epilogue]).  The
host does not synchronise inside the loop unless it must: ``t_final``
termination, an ``observer`` or a host ``dt_provider``.  Step records are
collected in HBM and read once at the end.  Invalid states latched by any
kernel are raised as the reference's ``StepError(step, stage)`` /
``InvalidStateError`` (timeint.py:161-165, 238-241).
"""

from __future__ import annotations

import os
import time as _time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .errors import InvalidStateError, StepError
from .grid import FieldSet, GridSpec, Layout, PeriodicHalo
from .physics import DEFAULT_PARAMS, GasModel, WenoParams
from .plan import error_from_key, get_plan
from .upwind import hyperbolic_rhs
from .viscous import parabolic_rhs

SCHEMES = ("rk3", "rk4")
CFL_MODES = ("max", "sum")
_SCHEME_CODE = {"rk3": _lib.HD_SCHEME_RK3, "rk4": _lib.HD_SCHEME_RK4}


@dataclass(frozen=True)
class TimeParams:
    """Scheme, step-size rule (fixed dt XOR CFL) and stop condition (timeint.py:38-65)."""

    scheme: str = "rk3"
    dt: float | None = None
    cfl: float | None = None
    cfl_mode: str = "max"
    t_final: float | None = None
    max_steps: int | None = None

    def __post_init__(self):
        if self.scheme not in SCHEMES:
            raise ValueError(f"scheme must be one of {SCHEMES}, got {self.scheme!r}")
        if self.cfl_mode not in CFL_MODES:
            raise ValueError(f"cfl_mode must be one of {CFL_MODES}, got {self.cfl_mode!r}")
        if (self.dt is None) == (self.cfl is None):
            raise ValueError("exactly one of dt and cfl must be set")
        if self.dt is not None and self.dt <= 0.0:
            raise ValueError(f"dt must be positive, got {self.dt}")
        if self.cfl is not None and self.cfl <= 0.0:
            raise ValueError(f"cfl must be positive, got {self.cfl}")
        if self.t_final is None and self.max_steps is None:
            raise ValueError("need a stop condition: t_final and/or max_steps")
        if self.t_final is not None and self.t_final < 0.0:
            raise ValueError(f"t_final must be nonnegative, got {self.t_final}")
        if self.max_steps is not None and self.max_steps < 0:
            raise ValueError(f"max_steps must be nonnegative, got {self.max_steps}")


@dataclass
class StepRecord:
    """Diagnostics of one completed step (timeint.py:68-86)."""

    step: int
    t: float
    dt: float
    mass: float
    momentum: tuple
    energy: float
    max_wavespeed: float
    wall_seconds: float
    kinetic_energy: float = float("nan")  # 0.5 <|m/rho|^2>: compute_spectrum().total() by Parseval
    enstrophy: float = float("nan")  # 0.5 <|curl(m/rho)|^2>, 4th-order central differences

    def log_line(self) -> str:
        mx, my, mz = self.momentum
        return (
            f"{self.step} {self.t:.12e} {self.dt:.12e} {self.mass:.15e} "
            f"{mx:.15e} {my:.15e} {mz:.15e} {self.energy:.15e} {self.wall_seconds:.6e}"
        )


@dataclass
class AdvanceResult:
    fields: FieldSet
    t: float
    records: list = field(default_factory=list)

    @property
    def steps(self) -> int:
        return len(self.records)


def _as_device(fields) -> FieldSet:
    """Device FieldSet for a device/host FieldSet or a reference (numpy) FieldSet.
    Host torch buffers (ideally pinned) are uploaded with one async copy."""
    if isinstance(fields, FieldSet):
        if fields.data.is_cuda:
            return fields
        dev = torch.device("cuda", torch.cuda.current_device())
        return FieldSet(fields.spec, fields.layout, fields.data.to(dev, non_blocking=True))
    return FieldSet.from_numpy(fields)


def _coerce(fields) -> FieldSet:
    """A FieldSet of this package (reference FieldSets are wrapped, not moved)."""
    return fields if isinstance(fields, FieldSet) else FieldSet.from_numpy(fields)


def _reduce(fields: FieldSet, gas: GasModel, tag: int = 0) -> np.ndarray:
    plan = get_plan(fields.spec, gas)
    out = torch.empty(_lib.HD_RED_N, dtype=torch.float64, device=fields.data.device)
    plan.reduce(fields.data, out, tag)
    vals = out.cpu().numpy()
    plan.raise_if_error(wrap_steps=False)
    return vals


def conserved_totals(fields: FieldSet, gas: GasModel = GasModel()):
    """Volume-weighted interior sums of mass, momentum and energy (timeint.py:100-107)."""
    r = _reduce(_as_device(fields), gas)
    vol = fields.spec.cell_volume()
    return (float(r[_lib.HD_RED_MASS]) * vol,
            tuple(float(r[_lib.HD_RED_MOMX + d]) * vol for d in range(3)),
            float(r[_lib.HD_RED_ENERGY]) * vol)


def max_wavespeed_interior(fields: FieldSet, gas: GasModel) -> float:
    """max over interior points and dimensions of |v_d| + a (timeint.py:115-119)."""
    return float(_reduce(_as_device(fields), gas)[_lib.HD_RED_WAVESPEED])


def kinetic_energy(fields: FieldSet, gas: GasModel = GasModel()) -> float:
    """Mean 0.5|m/rho|^2 over the interior = hit.compute_spectrum(...).total()."""
    r = _reduce(_as_device(fields), gas)
    return float(r[_lib.HD_RED_KE]) / fields.spec.interior_points


def enstrophy(fields: FieldSet, gas: GasModel = GasModel()) -> float:
    """Mean 0.5|curl v|^2 over the interior, v = m * (1/rho) (physics.py:249-252),
    each derivative the reference's central_derivative_4 (viscous.py:23-51).
    Refills the ghost layers of ``fields`` first (periodic), like the rhs does."""
    fs = _as_device(fields)
    plan = get_plan(fs.spec, gas)
    plan.fill_ghosts(fs.data, 5)
    out = torch.empty(1, dtype=torch.float64, device=fs.data.device)
    plan.enstrophy(fs.data, out)
    return float(out.item()) / fs.spec.interior_points


def max_signal(fields: FieldSet, gas: GasModel, cfl_mode: str = "max") -> float:
    """Largest per-point CFL signal (timeint.py:122-131)."""
    r = _reduce(_as_device(fields), gas)
    return float(r[_lib.HD_RED_SIGNAL_SUM if cfl_mode == "sum" else _lib.HD_RED_SIGNAL_MAX])


def compute_dt(fields: FieldSet, gas: GasModel, cfl: float, cfl_mode: str = "max") -> float:
    """cfl / max_signal; raises on a silent or non-finite field (timeint.py:133-138)."""
    signal = max_signal(fields, gas, cfl_mode)
    if not np.isfinite(signal) or signal <= 0.0:
        raise InvalidStateError(f"cannot size dt: max signal is {signal}")
    return cfl / signal


def make_rhs(gas: GasModel, params: WenoParams = DEFAULT_PARAMS, delta: float = 0.0, halo=None,
             workers: int = 1, mode: str | None = None):
    """rhs(u) = sync_ghosts(u); hyperbolic_rhs(u) + parabolic_rhs(u) (timeint.py:141-158)."""
    if halo is None:
        halo = PeriodicHalo()

    def rhs(fields: FieldSet) -> FieldSet:
        fields = _as_device(fields)
        halo.sync_fields(fields)
        inc = hyperbolic_rhs(fields, gas, params, delta, workers, mode=mode)
        parabolic_rhs(fields, gas, halo, workers, out=inc, mode=mode)
        return inc

    # the steppers recognise this closure and run the fused device step instead
    rhs.hd_config = (gas, params, float(delta), halo, mode)
    return rhs


def _stage(rhs, fields, stage: int):
    try:
        return rhs(fields)
    except InvalidStateError as err:
        raise StepError(f"invalid state entering RK stage {stage}: {err}", stage=stage) from err


def _fused_step(fields: FieldSet, dt: float, rhs, scheme: str) -> FieldSet:
    gas, params, delta, halo, mode = rhs.hd_config
    plan = get_plan(fields.spec, gas, params, delta, mode)
    out = fields.copy()
    dt_dev = torch.full((1,), float(dt), dtype=torch.float64, device=out.data.device)
    plan.step(_SCHEME_CODE[scheme], out.data, dt_dev, 0)
    key = plan.error_key()
    if key:
        from .plan import decode_key, error_from_key

        plan.error_clear()
        _, slot, _, _ = decode_key(key)
        err = error_from_key(key, fields.spec, wrap_steps=False)
        raise StepError(f"invalid state entering RK stage {slot - 1}: {err}", stage=slot - 1) from err
    return out


def _fusable(rhs, fields) -> bool:
    cfg = getattr(rhs, "hd_config", None)
    return (cfg is not None and isinstance(cfg[3], PeriodicHalo)
            and fields.layout == Layout.COMPONENT_CONTIGUOUS)


def rk3_tvd_step(fields: FieldSet, dt: float, rhs) -> FieldSet:
    """One three-stage TVD Runge-Kutta step (timeint.py:168-178).

    With a ``make_rhs`` closure the whole step is one fused device call; any
    other rhs callable is composed stage by stage like the reference (torch
    arithmetic on whatever device ``fields`` lives on)."""
    fields = _coerce(fields)
    if _fusable(rhs, fields):
        return _fused_step(_as_device(fields), dt, rhs, "rk3")
    spec, layout = fields.spec, fields.layout
    r0 = _stage(rhs, fields, 0)
    u1 = FieldSet(spec, layout, fields.data + dt * r0.data)
    r1 = _stage(rhs, u1, 1)
    u2 = FieldSet(spec, layout, 0.75 * fields.data + 0.25 * (u1.data + dt * r1.data))
    r2 = _stage(rhs, u2, 2)
    return FieldSet(spec, layout, (1.0 / 3.0) * fields.data + (2.0 / 3.0) * (u2.data + dt * r2.data))


def rk4_step(fields: FieldSet, dt: float, rhs) -> FieldSet:
    """One classical four-stage Runge-Kutta step (timeint.py:181-193); see rk3_tvd_step."""
    fields = _coerce(fields)
    if _fusable(rhs, fields):
        return _fused_step(_as_device(fields), dt, rhs, "rk4")
    spec, layout = fields.spec, fields.layout
    half = 0.5 * dt
    k1 = _stage(rhs, fields, 0)
    k2 = _stage(rhs, FieldSet(spec, layout, fields.data + half * k1.data), 1)
    k3 = _stage(rhs, FieldSet(spec, layout, fields.data + half * k2.data), 2)
    k4 = _stage(rhs, FieldSet(spec, layout, fields.data + dt * k3.data), 3)
    return FieldSet(spec, layout,
                    fields.data + (dt / 6.0) * (k1.data + 2.0 * k2.data + 2.0 * k3.data + k4.data))


STEPPERS = {"rk3": rk3_tvd_step, "rk4": rk4_step}


class _Records:
    """Per-step diagnostics kept in HBM: [t, dt, red[0..8]] per row."""

    def __init__(self, device, cap: int):
        self.rows = torch.empty((max(cap, 1), 2 + _lib.HD_RED_N), dtype=torch.float64, device=device)
        self.n = 0

    def push(self, ctx: torch.Tensor, red: torch.Tensor) -> None:
        if self.n == self.rows.shape[0]:
            grown = torch.empty((2 * self.n, self.rows.shape[1]), dtype=torch.float64,
                                device=self.rows.device)
            grown[: self.n] = self.rows
            self.rows = grown
        self.rows[self.n, 0:2] = ctx[0:2]
        self.rows[self.n, 2:] = red
        self.n += 1


ENS_COL = 2 + _lib.HD_RED_ENSTROPHY  # enstrophy sum in a record row


def _record(step: int, row: np.ndarray, spec: GridSpec, wall: float, points: int) -> StepRecord:
    vol = spec.cell_volume()
    red = row[2:]
    return StepRecord(
        step=step, t=float(row[0]), dt=float(row[1]),
        mass=float(red[_lib.HD_RED_MASS]) * vol,
        momentum=tuple(float(red[_lib.HD_RED_MOMX + d]) * vol for d in range(3)),
        energy=float(red[_lib.HD_RED_ENERGY]) * vol,
        max_wavespeed=float(red[_lib.HD_RED_WAVESPEED]),
        wall_seconds=wall,
        kinetic_energy=float(red[_lib.HD_RED_KE]) / points,
        enstrophy=float(row[ENS_COL]) / points,
    )


def advance(fields, gas: GasModel, tparams: TimeParams, weno_params: WenoParams = DEFAULT_PARAMS,
            delta: float = 0.0, halo=None, workers: int = 1, t0: float = 0.0, observer=None,
            dt_provider=None, mode: str | None = None) -> AdvanceResult:
    """March until t_final and/or max_steps, collecting step records (timeint.py:199-258).

    ``fields`` may be a device FieldSet or a host (reference) FieldSet; the
    input is not modified except for its ghost layers (as the reference's
    rhs refills them in place).
    """
    uploaded = isinstance(fields, FieldSet) and not fields.data.is_cuda
    fields = _as_device(fields)
    if fields.layout != Layout.COMPONENT_CONTIGUOUS:
        raise ValueError("advance needs COMPONENT_CONTIGUOUS fields")
    if halo is not None and not isinstance(halo, PeriodicHalo):
        from .decomp import DistHalo

        if isinstance(halo, DistHalo):
            return halo.advance(fields, gas, tparams, weno_params, delta, t0, observer, dt_provider,
                                mode)
        raise TypeError(f"unsupported halo {type(halo).__name__}")
    plan = get_plan(fields.spec, gas, weno_params, delta, mode)
    # a freshly uploaded host state is ours to march in place (no second device copy)
    runner = _DeviceMarch(plan, fields, gas, tparams, t0, copy=not uploaded)
    return runner.run(observer, dt_provider)


class _DeviceMarch:
    """The fused single-device march shared by advance() and the decomposed driver."""

    def __init__(self, plan, fields: FieldSet, gas: GasModel, tparams: TimeParams, t0: float,
                 stepper=None, reducer=None, global_points: int | None = None, copy: bool = True,
                 error_combine=None, ghost_sync=None, sum_combine=None, protocol_check=None):
        self.plan = plan
        self.spec = fields.spec
        # interior points of the whole (possibly decomposed) domain: the KE mean
        self.points = global_points or fields.spec.interior_points
        self.gas = gas
        self.tp = tparams
        self.t0 = float(t0)
        self.out = fields.copy() if copy else fields
        dev = self.out.data.device
        self.ctx = plan.ctx
        self.ctx.zero_()
        self.ctx[_lib.HD_CTX_T] = self.t0
        self.red = torch.zeros(_lib.HD_RED_N, dtype=torch.float64, device=dev)
        self.scheme = _SCHEME_CODE[tparams.scheme]
        # multi-rank drivers override how a step runs and how reductions combine
        self.own_stepper = stepper is None and reducer is None
        scheme = self.scheme  # the default stepper must not capture self (a reference cycle
        # would keep the plan's workspace alive until the next garbage collection)
        self.stepper = stepper or (lambda u, dt_dev, tag: plan.step(scheme, u, dt_dev, tag))
        self.reducer = reducer or (lambda red: None)
        self.error_combine = error_combine or (lambda key: key)
        # ghosts of the march state valid again after the last step (decomposed runs:
        # the final halo), and the rank sum of per-rank partial sums
        self.ghost_sync = ghost_sync or (lambda u: None)
        self.sum_combine = sum_combine or (lambda t: None)
        # decomposed runs: raise a halo failure (peer timeout) before the error keys it caused
        self.protocol_check = protocol_check or (lambda: None)

    def _enstrophy_now(self, dst: torch.Tensor) -> None:
        """Enstrophy sum of the current state into ``dst`` (one element)."""
        self.ghost_sync(self.out.data)
        self.plan.enstrophy(self.out.data, dst)

    def _reduce(self, tag: int) -> None:
        self.plan.reduce(self.out.data, self.red, tag)
        self.reducer(self.red)

    # steps per CUDA graph replay (the launch-bound small-grid path)
    GRAPH_CHUNK = 8
    # measured on B200 (tools/small_grid.py, 41 RK4 steps incl. capture): 32^3 0.52 -> 0.40
    # ms/step with graphs; 64^3 0.57 -> 0.62 and 128^3 2.39 -> 2.58 (kernel time dominates
    # there and the capture does not pay back)
    GRAPH_MAX_POINTS = 48 ** 3

    def _graph_ok(self, observer, dt_provider) -> bool:
        tp = self.tp
        env = os.environ.get("HD_NO_GRAPH")
        if env not in (None, "") and env != "0":
            return False
        small = self.spec.interior_points <= self.GRAPH_MAX_POINTS or env == "0"
        return (self.own_stepper and observer is None and dt_provider is None and tp.t_final is None
                and tp.max_steps is not None and tp.max_steps >= 1 + 2 * self.GRAPH_CHUNK
                and self.out.data.is_cuda and small)

    def _one_step(self, k: int, tag: int, cfl_mode: int) -> None:
        """Step k of the march: dt, the RK stages, time, diagnostics of the new state.
        ``tag`` is the step number the kernels latch errors with."""
        tp, plan = self.tp, self.plan
        if tp.dt is not None:
            plan.set_dt(None, 0, 0.0, tp.dt, -1.0, self.ctx, tag * 8)
        else:
            plan.set_dt(self.red, cfl_mode, tp.cfl, 0.0, -1.0, self.ctx, tag * 8)
        plan.arm_reduce(self.red, tag * 8 + 7)  # diagnostics of the new state (= next CFL signal)
        self.stepper(self.out.data, self.ctx[_lib.HD_CTX_DT:], tag)
        plan.commit_time(self.ctx)
        self.reducer(self.red)

    def _run_graph(self) -> AdvanceResult:
        """max_steps without host synchronisation, the steps replayed from CUDA
        graphs of GRAPH_CHUNK steps (one launch per chunk instead of ~23 per
        step).  Step 0 runs eagerly (it also loads every kernel); the kernels of
        a chunk latch errors with chunk-relative step tags, so the error key is
        moved to a per-chunk slot after each replay and decoded with the chunk's
        first step as the base (earliest step still wins)."""
        tp, plan = self.tp, self.plan
        plan.error_clear()
        dev = self.out.data.device
        cfl_mode = 1 if tp.cfl_mode == "sum" else 0
        S = self.GRAPH_CHUNK
        nsteps = tp.max_steps
        nchunks = (nsteps - 1) // S
        rows = torch.empty((nsteps, 2 + _lib.HD_RED_N), dtype=torch.float64, device=dev)
        err = plan.err_key
        slots = torch.full((nchunks + 1,), -1, dtype=torch.int64, device=dev)
        wall0 = _time.perf_counter()

        def record(k):
            rows[k, 0:2] = self.ctx[0:2]
            rows[k, 2:] = self.red
            plan.enstrophy(self.out.data, rows[k, ENS_COL:ENS_COL + 1])

        if tp.dt is None:
            self._reduce(0)
        self._one_step(0, 0, cfl_mode)
        record(0)
        slots[0] = err[0]
        err.fill_(-1)
        chunk_rows = torch.empty((S, 2 + _lib.HD_RED_N), dtype=torch.float64, device=dev)
        graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.graph(graph, stream=side):
            for r in range(S):
                self._one_step(1 + r, r, cfl_mode)
                chunk_rows[r, 0:2] = self.ctx[0:2]
                chunk_rows[r, 2:] = self.red
                plan.enstrophy(self.out.data, chunk_rows[r, ENS_COL:ENS_COL + 1])
        torch.cuda.current_stream(dev).wait_stream(side)
        for c in range(nchunks):
            graph.replay()
            rows[1 + c * S: 1 + (c + 1) * S] = chunk_rows
            slots[c + 1] = err[0]
            err.fill_(-1)
        for k in range(1 + nchunks * S, nsteps):
            self._one_step(k, k, cfl_mode)
            record(k)
        keys = slots.cpu().tolist()
        host_rows = rows.cpu().numpy()
        del graph
        for i, key in enumerate(keys):
            if key != -1:
                plan.error_clear()
                raise error_from_key(key & (2 ** 64 - 1), self.spec, 0 if i == 0 else 1 + (i - 1) * S)
        self._check(step_base=0)
        per = (_time.perf_counter() - wall0) / nsteps
        records = [_record(k + 1, host_rows[k], self.spec, per, self.points) for k in range(nsteps)]
        return AdvanceResult(fields=self.out, t=float(host_rows[-1][0]), records=records)

    def run(self, observer=None, dt_provider=None) -> AdvanceResult:
        if self._graph_ok(observer, dt_provider):
            return self._run_graph()
        tp, plan = self.tp, self.plan
        plan.error_clear()
        cap = tp.max_steps if tp.max_steps is not None else 64
        recs = _Records(self.out.data.device, cap)
        t_final = tp.t_final if tp.t_final is not None else -1.0
        time_tol = 1e-12 * max(1.0, abs(tp.t_final)) if tp.t_final is not None else 0.0
        sync_each = tp.t_final is not None or observer is not None or dt_provider is not None
        cfl_mode = 1 if tp.cfl_mode == "sum" else 0
        records: list[StepRecord] = []
        walls: list[float] = []
        t = self.t0
        step = 0
        have_signal = False
        last_wall = _time.perf_counter()
        while True:
            if tp.max_steps is not None and step >= tp.max_steps:
                break
            if tp.t_final is not None and t >= tp.t_final - time_tol:
                break
            wall0 = _time.perf_counter()
            tag_pre = step * 8
            if tp.dt is not None:
                plan.set_dt(None, 0, 0.0, tp.dt, t_final, self.ctx, tag_pre)
            elif dt_provider is not None:
                dt = float(dt_provider(self.out))
                plan.set_dt(None, 0, 0.0, dt, t_final, self.ctx, tag_pre)
            else:
                if not have_signal:
                    self._reduce(tag_pre)
                plan.set_dt(self.red, cfl_mode, tp.cfl, 0.0, t_final, self.ctx, tag_pre)
            # diagnostics of the new state (= next step's CFL signal), fused into the last
            # RK stage's update kernel when the plan can (hd_arm_reduce); the enstrophy of
            # the previous step's result, folded into this step's first flux kernel
            plan.arm_reduce(self.red, step * 8 + 7)
            if step >= 1 and not sync_each:
                plan.arm_enstrophy(recs.rows[step - 1, ENS_COL:ENS_COL + 1])
            self.stepper(self.out.data, self.ctx[_lib.HD_CTX_DT:], step)
            plan.commit_time(self.ctx)
            self.reducer(self.red)
            have_signal = True
            recs.push(self.ctx, self.red)
            step += 1
            if sync_each:
                ens = recs.rows[step - 1, ENS_COL:ENS_COL + 1]
                self._enstrophy_now(ens)
                self.sum_combine(ens)
                row = recs.rows[step - 1].cpu().numpy()
                self._check(step_base=0)
                t = float(row[0])
                wall = _time.perf_counter() - wall0
                rec = _record(step, row, self.spec, wall, self.points)
                records.append(rec)
                if observer is not None:
                    observer(rec)
        if not sync_each:
            if step:
                self._enstrophy_now(recs.rows[step - 1, ENS_COL:ENS_COL + 1])
                ens = recs.rows[: recs.n, ENS_COL].contiguous()
                self.sum_combine(ens)
                recs.rows[: recs.n, ENS_COL] = ens
            rows = recs.rows[: recs.n].cpu().numpy()
            self._check(step_base=0)
            total = _time.perf_counter() - last_wall
            per = total / max(step, 1)
            records = [_record(s + 1, rows[s], self.spec, per, self.points) for s in range(step)]
            if step:
                t = float(rows[step - 1][0])
        return AdvanceResult(fields=self.out, t=t, records=records)

    def _check(self, step_base: int) -> None:
        """Raise the latched error; multi-rank drivers combine the keys first
        (``error_combine``) so every rank raises the same error at the same step."""
        self.protocol_check()
        key = self.error_combine(self.plan.error_key())
        if key:
            self.plan.error_clear()
            raise error_from_key(key, self.spec, step_base)


def write_step_log(path, records) -> None:
    """`step t dt mass mom_x mom_y mom_z energy wall_seconds` (timeint.py:261-266)."""
    with open(path, "w") as fh:
        for rec in records:
            fh.write(rec.log_line() + "\n")
