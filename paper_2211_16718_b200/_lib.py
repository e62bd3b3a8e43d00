"""ctypes binding of libhd.so (the C ABI declared in include/hd.h).

The product path has exactly one implementation: the sm_100a kernels in
``csrc/``.  There is no CPU fallback -- if the shared library is missing, or
no CUDA device is present, every compute entry point raises
:class:`NativeUnavailable`.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HD_LIB") or os.path.join(HERE, "libhd.so")
CSRC = os.path.join(HERE, "csrc")

HD_OK = 0
HD_E_ARG, HD_E_CUDA, HD_E_WORKSPACE, HD_E_UNSUPPORTED = -1, -2, -3, -4
HD_MODE_FAST = 0
HD_MODE_EXACT = 1
HD_SCHEME_RK3 = 3
HD_SCHEME_RK4 = 4
HD_PART_LOCAL, HD_PART_HALO, HD_PART_MID, HD_PART_UPDATE, HD_PART_ALL = 1, 2, 4, 8, 15
HD_OPT_SEGMENTS, HD_OPT_X_STAGED, HD_OPT_FLUX_ZMARCH, HD_OPT_FLUX_TMA, HD_OPT_SWEEP_WAVES = 0, 1, 2, 3, 4
(HD_BUF_STAGE, HD_BUF_ACC, HD_BUF_INC, HD_BUF_PRIM, HD_BUF_VFLUX, HD_BUF_RED, HD_BUF_CTX,
 HD_BUF_ERR, HD_BUF_STATE, HD_BUF_SYNC, HD_BUF_FRED, HD_BUF_ENS) = range(12)
HD_PEER_STATE, HD_PEER_VFLUX = 0, 1
(HD_RED_SIGNAL_MAX, HD_RED_SIGNAL_SUM, HD_RED_WAVESPEED, HD_RED_MASS, HD_RED_MOMX, HD_RED_MOMY,
 HD_RED_MOMZ, HD_RED_ENERGY, HD_RED_KE, HD_RED_ENSTROPHY) = range(10)
HD_RED_N = 10
HD_CTX_T, HD_CTX_DT = 0, 1
HD_CTX_N = 4

# every symbol include/hd.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "hd_abi_version", "hd_status_string", "hd_workspace_bytes", "hd_plan_create",
    "hd_plan_destroy", "hd_plan_set_option", "hd_plan_buffer", "hd_plan_total_points", "hd_fill_ghosts",
    "hd_hyper_sweep", "hd_hyperbolic_rhs", "hd_parabolic_rhs", "hd_central_diff4", "hd_rhs",
    "hd_step", "hd_stage_part", "hd_reduce_state", "hd_set_dt", "hd_commit_time",
    "hd_error_read", "hd_error_clear", "hd_fp64_probe", "hd_bench_weights", "hd_launch_counter", "hd_timer_enable",
    "hd_timer_read", "hd_ipc_handle", "hd_ipc_open", "hd_ipc_close", "hd_peer_attach", "hd_peer_attach3", "hd_peer_signal",
    "hd_peer_wait", "hd_peer_timed_out", "hd_stage_buffer", "hd_rk4_step", "hd_max_signal",
    "hd_totals", "hd_error_flags", "hd_halo_exchange", "hd_viscous_fluxes", "hd_viscous_divergence",
    "hd_arm_reduce", "hd_enstrophy", "hd_arm_enstrophy", "hd_hyper_sweep_lines",
)
# hd_timer_read kinds (HD_TK_*)
TIMER_KINDS = ("sweep_x", "sweep_y", "sweep_z", "gradflux", "prims", "divergence", "reduce")


class NativeUnavailable(RuntimeError):
    """libhd.so (the only implementation of the hot path) cannot run here."""


class HdError(RuntimeError):
    """A libhd call returned a negative status."""


class HdGeom(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int * 3),
        ("length", ctypes.c_double * 3),
        ("ghost", ctypes.c_int),
        ("periodic", ctypes.c_int * 3),
    ]


class HdGas(ctypes.Structure):
    _fields_ = [("gamma", ctypes.c_double), ("prandtl", ctypes.c_double),
                ("mu", ctypes.c_double), ("visc_scale", ctypes.c_double)]


class HdWeno(ctypes.Structure):
    _fields_ = [("epsilon", ctypes.c_double), ("power", ctypes.c_int), ("delta", ctypes.c_double)]


_lib = None


def build(force: bool = False) -> str:
    """Compile libhd.so in-tree with nvcc for sm_100a (make -C csrc)."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-s", "-C", CSRC, "-j4"], check=True)
    return LIB_PATH


def load(require_cuda: bool = False):
    """Load libhd.so and declare the ABI; no compute happens here."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(f"{LIB_PATH} is not built; run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        i32, i64, f64 = ctypes.c_int, ctypes.c_int64, ctypes.c_double
        sig = {
            "hd_abi_version": ([], i32),
            "hd_status_string": ([i32], ctypes.c_char_p),
            "hd_workspace_bytes": ([ctypes.POINTER(HdGeom)], i64),
            "hd_plan_create": ([ctypes.POINTER(HdGeom), ctypes.POINTER(HdGas), ctypes.POINTER(HdWeno),
                                i32, P, i64, ctypes.POINTER(P)], i32),
            "hd_plan_destroy": ([P], i32),
            "hd_plan_buffer": ([P, i32], P),
            "hd_plan_total_points": ([P], i64),
            "hd_fill_ghosts": ([P, P, i32, P], i32),
            "hd_hyper_sweep": ([P, i32, P, P, i32, P], i32),
            "hd_hyperbolic_rhs": ([P, P, P, i32, P], i32),
            "hd_parabolic_rhs": ([P, P, P, P], i32),
            "hd_central_diff4": ([P, P] + [i32] * 10 + [f64, P], i32),
            "hd_rhs": ([P, P, P, P], i32),
            "hd_step": ([P, i32, P, P, i64, P], i32),
            "hd_plan_set_option": ([P, i32, i64], i32),
            "hd_stage_part": ([P, i32, i32, i32, P, P, i64, P], i32),
            "hd_reduce_state": ([P, P, P, i64, P], i32),
            "hd_set_dt": ([P, P, i32, f64, f64, f64, P, i64, P], i32),
            "hd_commit_time": ([P, P, P], i32),
            "hd_error_read": ([P, ctypes.POINTER(ctypes.c_uint64), P], i32),
            "hd_error_clear": ([P, P], i32),
            "hd_fp64_probe": ([P, i32, i32, i32, P], i32),
            "hd_bench_weights": ([P, i32, i32, i32, i32, i32, i32, i32, i32, ctypes.c_double, i32, P,
                                  ctypes.POINTER(ctypes.c_int64), P], i32),
            "hd_launch_counter": ([], i64),
            "hd_stage_buffer": ([P, i32, i32, P, ctypes.POINTER(ctypes.c_void_p)], i32),
            "hd_rk4_step": ([P, P, P, P], i32),
            "hd_arm_reduce": ([P, P, i64], i32),
            "hd_enstrophy": ([P, P, P, P], i32),
            "hd_hyper_sweep_lines": ([P, P, P] + [i64] * 9 + [i32, f64, f64, f64, i32, f64, P], i32),
            "hd_arm_enstrophy": ([P, P], i32),
            "hd_viscous_fluxes": ([P, P, P], i32),
            "hd_viscous_divergence": ([P, P, P], i32),
            "hd_max_signal": ([P, P, P, i32, P], i32),
            "hd_totals": ([P, P, P, P], i32),
            "hd_error_flags": ([P, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int64), P], i32),
            "hd_halo_exchange": ([P, P, i32, P], i32),
            "hd_ipc_handle": ([P, P, ctypes.POINTER(ctypes.c_int64)], i32),
            "hd_ipc_open": ([P, i64, ctypes.POINTER(ctypes.c_void_p)], i32),
            "hd_ipc_close": ([P, i64], i32),
            "hd_peer_attach": ([P, P, P, P], i32),
            "hd_peer_attach3": ([P, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p), P], i32),
            "hd_peer_signal": ([P, i32, i64, P], i32),
            "hd_peer_wait": ([P, i32, i64, P], i32),
            "hd_peer_timed_out": ([P, ctypes.POINTER(ctypes.c_int), P], i32),
            "hd_timer_enable": ([P, i32], i32),
            "hd_timer_read": ([P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64), i32],
                              i32),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    if require_cuda:
        import torch

        if not torch.cuda.is_available():
            raise NativeUnavailable("no CUDA device: the hitdns hot path only runs on the GPU")
    return _lib


def check(status: int, what: str = "") -> None:
    if status != HD_OK:
        msg = load().hd_status_string(status).decode()
        raise HdError(f"{what}: libhd status {status} ({msg})")
