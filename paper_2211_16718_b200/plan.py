"""Device plans: one ``hd_plan`` (include/hd.h) per geometry/physics/mode.

A :class:`Plan` owns its HBM workspace as a torch tensor (stage state, RK4
accumulator, RHS increment, 4 primitive and 12 viscous-flux fields, reduction
partials, step context, error key) and exposes the C ABI as methods that
launch on the current torch CUDA stream.  Plans are cached per key; a 512^3
plan holds ~34 GB, so the cache is small and :func:`release_plans` drops it.
"""

from __future__ import annotations

import ctypes
import gc
import os
from collections import OrderedDict

import torch

from . import _lib
from .errors import InvalidStateError, StepError
from .grid import GridSpec
from .physics import DEFAULT_PARAMS, GasModel, WenoParams

_MODES = {"fast": _lib.HD_MODE_FAST, "exact": _lib.HD_MODE_EXACT}
_mode = os.environ.get("HD_MODE", "fast").lower()
if _mode not in _MODES:
    _mode = "fast"


def set_mode(mode: str) -> None:
    """Select the arithmetic mode of new plans: "fast" (default) or "exact"
    (reference operation order, bitwise equal to the reference)."""
    global _mode
    if mode not in _MODES:
        raise ValueError(f"mode must be one of {tuple(_MODES)}, got {mode!r}")
    _mode = mode


def get_mode() -> str:
    return _mode


def _stream_ptr() -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t: torch.Tensor) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


class Plan:
    """An hd_plan plus its workspace on the current CUDA device."""

    def __init__(self, spec: GridSpec, gas: GasModel = GasModel(), weno: WenoParams = DEFAULT_PARAMS,
                 delta: float = 0.0, mode: str | None = None, periodic=(True, True, True),
                 workspace: bool = True):
        L = _lib.load(require_cuda=True)
        self.L = L
        self.spec = spec
        self.gas, self.weno, self.delta = gas, weno, float(delta)
        self.mode = mode or _mode
        self.periodic = tuple(bool(p) for p in periodic)
        g = _lib.HdGeom()
        for d in range(3):
            g.n[d] = spec.n[d]
            g.length[d] = spec.length[d]
            g.periodic[d] = 1 if self.periodic[d] else 0
        g.ghost = spec.ghost_width
        self._geom = g
        gs = _lib.HdGas(gas.gamma, gas.prandtl, gas.mu, gas.visc_scale)
        wp = _lib.HdWeno(weno.epsilon, weno.power, self.delta)
        self.device = torch.device("cuda", torch.cuda.current_device())
        self.ws = None
        nbytes = 0
        if workspace:
            nbytes = int(L.hd_workspace_bytes(ctypes.byref(g)))
            if nbytes < 0:
                _lib.check(nbytes, "hd_workspace_bytes")
            self.ws = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
            base = self.ws.data_ptr()
            self._ws_off = (-base) % 256
            ws_ptr = ctypes.c_void_p(base + self._ws_off)
        else:
            ws_ptr = ctypes.c_void_p(None)
        h = ctypes.c_void_p()
        _lib.check(L.hd_plan_create(ctypes.byref(g), ctypes.byref(gs), ctypes.byref(wp),
                                    _MODES[self.mode], ws_ptr, nbytes, ctypes.byref(h)),
                   "hd_plan_create")
        self.h = h
        self.npts = spec.total_points
        self._bufs = {}
        waves = os.environ.get("HD_SWEEP_WAVES")  # tuning knob, read once per plan
        if waves:
            self.set_option(_lib.HD_OPT_SWEEP_WAVES, int(waves))

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            try:
                self.L.hd_plan_destroy(h)
            except Exception:  # noqa: BLE001 - interpreter shutdown
                pass
            self.h = None

    # ---- workspace views ------------------------------------------------
    def buffer(self, which: int, count: int) -> torch.Tensor:
        """fp64 view of workspace buffer ``which`` (count doubles)."""
        key = (which, count)
        if key not in self._bufs:
            ptr = self.L.hd_plan_buffer(self.h, which)
            off = ptr - self.ws.data_ptr()
            self._bufs[key] = self.ws[off: off + 8 * count].view(torch.float64)
        return self._bufs[key]

    def fields(self, which: int, nfields: int) -> torch.Tensor:
        return self.buffer(which, nfields * self.npts)

    @property
    def ctx(self) -> torch.Tensor:
        return self.buffer(_lib.HD_BUF_CTX, _lib.HD_CTX_N)

    @property
    def err_key(self) -> torch.Tensor:
        """The device error key (int64 view; -1 = none)."""
        key = ("err", 1)
        if key not in self._bufs:
            ptr = self.L.hd_plan_buffer(self.h, _lib.HD_BUF_ERR)
            off = ptr - self.ws.data_ptr()
            self._bufs[key] = self.ws[off: off + 8].view(torch.int64)
        return self._bufs[key]

    @property
    def red(self) -> torch.Tensor:
        """Slot for the HD_RED_* results (after the partials)."""
        full = self.buffer(_lib.HD_BUF_RED, 2048 * 9 + 16)
        return full[2048 * 9: 2048 * 9 + _lib.HD_RED_N]

    # ---- C ABI ----------------------------------------------------------
    def fill_ghosts(self, t: torch.Tensor, nfields: int) -> None:
        _lib.check(self.L.hd_fill_ghosts(self.h, _ptr(t), nfields, _stream_ptr()), "hd_fill_ghosts")

    def hyper_sweep(self, dim: int, u, inc, accumulate: bool = True) -> None:
        _lib.check(self.L.hd_hyper_sweep(self.h, dim, _ptr(u), _ptr(inc), int(accumulate),
                                         _stream_ptr()), "hd_hyper_sweep")

    def hyperbolic_rhs(self, u, inc, accumulate: bool) -> None:
        _lib.check(self.L.hd_hyperbolic_rhs(self.h, _ptr(u), _ptr(inc), int(accumulate),
                                            _stream_ptr()), "hd_hyperbolic_rhs")

    def parabolic_rhs(self, u, inc) -> None:
        _lib.check(self.L.hd_parabolic_rhs(self.h, _ptr(u), _ptr(inc), _stream_ptr()),
                   "hd_parabolic_rhs")

    def rhs(self, u, inc) -> None:
        _lib.check(self.L.hd_rhs(self.h, _ptr(u), _ptr(inc), _stream_ptr()), "hd_rhs")

    def step(self, scheme: int, u, dt_dev, tag: int) -> None:
        _lib.check(self.L.hd_step(self.h, scheme, _ptr(u), _ptr(dt_dev), tag, _stream_ptr()), "hd_step")

    def set_option(self, option: int, value: int) -> None:
        """Kernel selection (HD_OPT_*): sweep segments per line, staged x sweep,
        z-marching flux kernel.  The state and dt never depend on it (the fused
        diagnostics' summation order follows the z sweep's segmentation)."""
        _lib.check(self.L.hd_plan_set_option(self.h, option, int(value)), "hd_plan_set_option")

    def stage_part(self, scheme: int, stage: int, parts: int, u, dt_dev, tag: int) -> None:
        _lib.check(self.L.hd_stage_part(self.h, scheme, stage, parts, _ptr(u),
                                        _ptr(dt_dev) if dt_dev is not None else ctypes.c_void_p(None),
                                        tag, _stream_ptr()), "hd_stage_part")

    def reduce(self, u, out, tag: int) -> None:
        _lib.check(self.L.hd_reduce_state(self.h, _ptr(u), _ptr(out), tag, _stream_ptr()),
                   "hd_reduce_state")

    def arm_reduce(self, out, tag: int) -> None:
        """The next completed step also writes the diagnostics of its result to
        ``out`` (fused into the last z sweep in fast mode; hd_arm_reduce)."""
        _lib.check(self.L.hd_arm_reduce(self.h, _ptr(out), tag), "hd_arm_reduce")

    def enstrophy(self, u, out) -> None:
        """out[0] = sum over the interior of 0.5 |curl(m/rho)|^2 (ghosts of u valid)."""
        _lib.check(self.L.hd_enstrophy(self.h, _ptr(u), _ptr(out), _stream_ptr()), "hd_enstrophy")

    def arm_enstrophy(self, out) -> None:
        """The next step also writes the enstrophy sum of its start state to ``out``
        (folded into the stage-0 viscous flux kernel; hd_arm_enstrophy)."""
        _lib.check(self.L.hd_arm_enstrophy(self.h, _ptr(out)), "hd_arm_enstrophy")

    def set_dt(self, red, cfl_mode: int, cfl: float, dt_fixed: float, t_final: float, ctx,
               tag: int) -> None:
        _lib.check(self.L.hd_set_dt(self.h, _ptr(red) if red is not None else ctypes.c_void_p(None),
                                    cfl_mode, cfl, dt_fixed, t_final, _ptr(ctx), tag,
                                    _stream_ptr()), "hd_set_dt")

    def commit_time(self, ctx) -> None:
        _lib.check(self.L.hd_commit_time(self.h, _ptr(ctx), _stream_ptr()), "hd_commit_time")

    def timer_enable(self, on: bool = True) -> None:
        _lib.check(self.L.hd_timer_enable(self.h, int(on)), "hd_timer_enable")

    def timer_read(self) -> dict:
        """{kind: (total ms, launches)} since the last read (CUDA events around each launch)."""
        n = len(_lib.TIMER_KINDS)
        ms = (ctypes.c_double * n)()
        cnt = (ctypes.c_int64 * n)()
        _lib.check(self.L.hd_timer_read(self.h, ms, cnt, n), "hd_timer_read")
        return {k: (ms[i], cnt[i]) for i, k in enumerate(_lib.TIMER_KINDS)}

    def stage_input(self, scheme: int, stage: int, u: torch.Tensor) -> torch.Tensor:
        """The 5-field buffer RK stage ``stage`` reads (``u`` for stage 0)."""
        if stage == 0:
            return u
        out = ctypes.c_void_p()
        _lib.check(self.L.hd_stage_buffer(self.h, scheme, stage - 1, _ptr(u), ctypes.byref(out)),
                   "hd_stage_buffer")
        if out.value == u.data_ptr():
            return u
        off = out.value - self.ws.data_ptr()
        n = 5 * self.npts
        return self.ws[off: off + 8 * n].view(torch.float64)

    # ---- peer halo over NVLink (z slabs) ----------------------------------
    def ipc_handle(self) -> tuple:
        """(64-byte IPC handle, offset) of this plan's workspace for a z neighbour."""
        h = (ctypes.c_char * 64)()
        off = ctypes.c_int64(0)
        _lib.check(self.L.hd_ipc_handle(ctypes.c_void_p(self.ws.data_ptr() + self._ws_off), h,
                                        ctypes.byref(off)), "hd_ipc_handle")
        return bytes(h), int(off.value)

    def peer_attach(self, lo, hi) -> None:
        """Neighbours' workspace pointers per axis (None for an unsplit axis)."""
        lo3 = (ctypes.c_void_p * 3)(*[ctypes.c_void_p(p) for p in lo])
        hi3 = (ctypes.c_void_p * 3)(*[ctypes.c_void_p(p) for p in hi])
        _lib.check(self.L.hd_peer_attach3(self.h, lo3, hi3, _stream_ptr()), "hd_peer_attach3")

    def peer_signal(self, which: int, value: int) -> None:
        _lib.check(self.L.hd_peer_signal(self.h, which, value, _stream_ptr()), "hd_peer_signal")

    def peer_wait(self, which: int, value: int) -> None:
        _lib.check(self.L.hd_peer_wait(self.h, which, value, _stream_ptr()), "hd_peer_wait")

    def peer_timed_out(self) -> bool:
        out = ctypes.c_int(0)
        _lib.check(self.L.hd_peer_timed_out(self.h, ctypes.byref(out), _stream_ptr()),
                   "hd_peer_timed_out")
        return bool(out.value)

    def error_key(self) -> int:
        key = ctypes.c_uint64(0)
        _lib.check(self.L.hd_error_read(self.h, ctypes.byref(key), _stream_ptr()), "hd_error_read")
        return int(key.value)

    def error_clear(self) -> None:
        _lib.check(self.L.hd_error_clear(self.h, _stream_ptr()), "hd_error_clear")

    def raise_if_error(self, step_base: int = 0, wrap_steps: bool = True) -> None:
        """Map a latched device error to the reference exceptions
        (InvalidStateError -> StepError(step, stage), timeint.py:161-165, 238-241)."""
        key = self.error_key()
        if not key:
            return
        self.error_clear()
        raise error_from_key(key, self.spec, step_base, wrap_steps)


def decode_key(key: int):
    """(step, slot, code, point); slot 1..4 = RK stage slot-1, 0/7 = reductions."""
    tag = key >> 36
    code = (key >> 34) & 3
    point = key & ((1 << 34) - 1)
    return tag >> 3, tag & 7, code, point


def error_from_key(key: int, spec: GridSpec, step_base: int = 0, wrap_steps: bool = True):
    step, slot, code, point = decode_key(key)
    if code == 3:
        return InvalidStateError("cannot size dt: max signal is zero or not finite")
    stage = slot - 1
    g = spec.ghost_width
    gx, gy = spec.n[0] + 2 * g, spec.n[1] + 2 * g
    where = (point // (gx * gy), (point // gx) % gy, point % gx)  # (z, y, x) ghosted index
    if not (1 <= slot <= 4):
        # the CFL reduction / step diagnostics decode the interior only
        # (timeint.py:110-112 cons_to_prim on fields.interior()): interior index
        where = tuple(c - g for c in where)
    # RK stages: the first copy in C order over the filled ghosted box, as the
    # reference's decode_primitives reports it (kernels latch first_image)
    kind = "density" if code == 1 else "pressure"
    inner = InvalidStateError(f"nonpositive {kind} at array index {where}", where=where)
    if not (1 <= slot <= 4) or not wrap_steps:
        return inner
    err = StepError(f"invalid state entering RK stage {stage}: {inner}", stage=stage)
    err.__cause__ = inner
    outer = StepError(f"step {step_base + step + 1} failed: {err}", step=step_base + step + 1,
                      stage=stage)
    outer.__cause__ = err
    return outer


_cache: "OrderedDict[tuple, Plan]" = OrderedDict()
_geo_cache: "OrderedDict[tuple, Plan]" = OrderedDict()
MAX_PLANS = int(os.environ.get("HD_MAX_PLANS", "3"))


def get_plan(spec: GridSpec, gas: GasModel = GasModel(), weno: WenoParams = DEFAULT_PARAMS,
             delta: float = 0.0, mode: str | None = None, periodic=(True, True, True)) -> Plan:
    mode = mode or _mode
    key = (spec, gas, weno, float(delta), mode, tuple(bool(p) for p in periodic),
           torch.cuda.current_device() if torch.cuda.is_available() else -1)
    plan = _cache.get(key)
    if plan is None:
        while len(_cache) >= MAX_PLANS:
            _cache.popitem(last=False)
        plan = Plan(spec, gas, weno, delta, mode, periodic)
        _cache[key] = plan
    else:
        _cache.move_to_end(key)
    return plan


def geometry_plan(spec: GridSpec, periodic=(True, True, True)) -> Plan:
    """Workspace-free plan for ghost fills of arbitrary field counts."""
    key = (spec, tuple(periodic), torch.cuda.current_device() if torch.cuda.is_available() else -1)
    plan = _geo_cache.get(key)
    if plan is None:
        if len(_geo_cache) > 16:
            _geo_cache.popitem(last=False)
        plan = Plan(spec, periodic=periodic, workspace=False)
        _geo_cache[key] = plan
    return plan


def release_plans() -> None:
    _cache.clear()
    _geo_cache.clear()
    gc.collect()  # plans referenced only from reference cycles go now, not at the next collection
    if torch.cuda.is_available():
        torch.cuda.empty_cache()
