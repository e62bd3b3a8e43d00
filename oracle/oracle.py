"""ctypes front-end of the C oracle (hd_oracle.c) -- TEST INFRASTRUCTURE ONLY.

This module is the parity checker for the CUDA product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import it; the product package never does.

The functions mirror the reference hot-path entry points on plain numpy
buffers in the reference's own flat COMPONENT_CONTIGUOUS layout
(``var * total_points + point``, x fastest; pkg/src/hitdns/grid.py:12-17):

* :func:`hyper_sweep`      -- kernels.py:68-73 signature, bit-exact
* :func:`central_diff4`    -- kernels.py:207-208 signature, bit-exact
* :func:`rhs`              -- timeint.py:152-156 (ghost sync + hyperbolic + parabolic)
* :func:`rk4_step`         -- timeint.py:181-193
* :func:`rk3_step`         -- timeint.py:168-178
* :func:`max_signal`       -- timeint.py:122-131
* :func:`advance`          -- timeint.py:199-258 without diagnostics
* :func:`enstrophy`        -- 0.5 <|curl v|^2> from decode_primitives + central_derivative_4
* :func:`bench_weights`    -- kernels.py:243-291 (layout-study weight kernel), numpy

Parity of this oracle against the reference itself is pinned by
``tests/test_oracle_golden.py`` (fixtures from ``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)


class OracleGeom(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int * 3),
        ("length", ctypes.c_double * 3),
        ("g", ctypes.c_int),
        ("gamma", ctypes.c_double),
        ("prandtl", ctypes.c_double),
        ("mu_eff", ctypes.c_double),
        ("eps", ctypes.c_double),
        ("delta", ctypes.c_double),
        ("power", ctypes.c_int),
    ]


def build() -> str:
    """Compile liboracle.so in place (make); returns its path."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        i64 = ctypes.c_int64
        L.or_hyper_sweep.argtypes = [_dp, _dp, _dp, i64, i64, i64, i64, i64, i64, i64, i64, i64,
                                     ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                     ctypes.c_double, ctypes.c_int, ctypes.c_double]
        L.or_hyper_sweep.restype = None
        L.or_central_diff4.argtypes = [_dp, _dp] + [ctypes.c_int] * 10 + [ctypes.c_double]
        L.or_central_diff4.restype = None
        L.or_fill_ghosts.argtypes = [_dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.or_fill_ghosts.restype = None
        L.or_work_size.argtypes = [ctypes.POINTER(OracleGeom)]
        L.or_work_size.restype = i64
        for name in ("or_rhs",):
            getattr(L, name).argtypes = [ctypes.POINTER(OracleGeom), _dp, _dp, _dp, _i64p]
            getattr(L, name).restype = ctypes.c_int
        for name in ("or_rk4_step", "or_rk3_step"):
            getattr(L, name).argtypes = [ctypes.POINTER(OracleGeom), _dp, ctypes.c_double, _dp, _i64p]
            getattr(L, name).restype = ctypes.c_int
        L.or_max_signal.argtypes = [ctypes.POINTER(OracleGeom), _dp, ctypes.c_int, _dp, _i64p]
        L.or_max_signal.restype = ctypes.c_int
        L.or_advance.argtypes = [ctypes.POINTER(OracleGeom), _dp, ctypes.c_int, ctypes.c_double,
                                 ctypes.c_double, ctypes.c_int, _dp, _i64p]
        L.or_advance.restype = ctypes.c_int
        L.or_enstrophy.argtypes = [ctypes.POINTER(OracleGeom), _dp]
        L.or_enstrophy.restype = ctypes.c_double
        L.or_num_threads.argtypes = []
        L.or_num_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


class OracleStateError(ValueError):
    """Nonpositive density (code 1) or pressure (code 2) met by the oracle."""

    def __init__(self, code: int, where: int, stage: int | None = None, step: int | None = None):
        kind = {1: "density", 2: "pressure"}.get(code, f"code {code}")
        super().__init__(f"nonpositive {kind} at flat point {where}" +
                         (f" in stage {stage}" if stage is not None else "") +
                         (f" of step {step}" if step is not None else ""))
        self.code, self.where, self.stage, self.step = code, where, stage, step


@dataclass(frozen=True)
class Problem:
    """Geometry + physics of one oracle run (mirrors GridSpec/GasModel/WenoParams)."""

    n: tuple
    length: tuple = (2 * math.pi,) * 3
    g: int = 3
    gamma: float = 1.4
    prandtl: float = 0.72
    mu: float = 0.0
    visc_scale: float = 1.0
    eps: float = 1e-6
    power: int = 2
    delta: float = 0.0

    def geom(self) -> OracleGeom:
        G = OracleGeom()
        for d in range(3):
            G.n[d] = int(self.n[d])
            G.length[d] = float(self.length[d])
        G.g = self.g
        G.gamma, G.prandtl = self.gamma, self.prandtl
        G.mu_eff = self.mu * self.visc_scale
        G.eps, G.delta, G.power = self.eps, self.delta, self.power
        return G

    @property
    def npts(self) -> int:
        g = self.g
        return (self.n[0] + 2 * g) * (self.n[1] + 2 * g) * (self.n[2] + 2 * g)

    @property
    def shape(self):
        g = self.g
        return (self.n[2] + 2 * g, self.n[1] + 2 * g, self.n[0] + 2 * g)


def num_threads() -> int:
    return int(lib().or_num_threads())


def set_num_threads(n: int) -> None:
    """OpenMP threads of the oracle's loops (results are invariant to it)."""
    lib().or_set_num_threads(int(n))


def hyper_sweep(u, f, inc, npts, base0, sd, sa, sb, nd, nb, a_lo, a_hi, dim, inv_dx, gamma,
                eps, power, delta):
    """kernels.py:68-73 signature; accumulates into ``inc``."""
    lib().or_hyper_sweep(_p(u), _p(f), _p(inc), npts, base0, sd, sa, sb, nd, nb, a_lo, a_hi,
                         dim, inv_dx, gamma, eps, power, delta)


def central_diff4(src, dst, di, dj, dk, g, og, nx, ny, nz, k_lo, k_hi, coef):
    """kernels.py:207-208 signature; writes the interior of ``dst``."""
    lib().or_central_diff4(_p(src), _p(dst), di, dj, dk, g, og, nx, ny, nz, k_lo, k_hi, coef)


def fill_ghosts(u: np.ndarray, prob: Problem) -> np.ndarray:
    lib().or_fill_ghosts(_p(u), prob.n[0], prob.n[1], prob.n[2], prob.g)
    return u


def _work(prob: Problem, G: OracleGeom) -> np.ndarray:
    return np.empty(int(lib().or_work_size(ctypes.byref(G))))


def rhs(u: np.ndarray, prob: Problem) -> np.ndarray:
    """Ghost sync of ``u`` (in place) then hyperbolic + parabolic increment."""
    G = prob.geom()
    inc = np.empty_like(u)
    where = ctypes.c_int64(-1)
    rc = lib().or_rhs(ctypes.byref(G), _p(u), _p(inc), _p(_work(prob, G)), ctypes.byref(where))
    if rc:
        raise OracleStateError(rc, where.value)
    return inc


def _step(fn, u, dt, prob):
    G = prob.geom()
    where = ctypes.c_int64(-1)
    rc = fn(ctypes.byref(G), _p(u), float(dt), _p(_work(prob, G)), ctypes.byref(where))
    if rc:
        raise OracleStateError(rc % 10, where.value, stage=rc // 10)
    return u


def rk4_step(u: np.ndarray, dt: float, prob: Problem) -> np.ndarray:
    """One classical RK4 step, in place (timeint.py:181-193)."""
    return _step(lib().or_rk4_step, u, dt, prob)


def rk3_step(u: np.ndarray, dt: float, prob: Problem) -> np.ndarray:
    """One TVD-RK3 step, in place (timeint.py:168-178)."""
    return _step(lib().or_rk3_step, u, dt, prob)


def max_signal(u: np.ndarray, prob: Problem, cfl_mode: str = "max") -> tuple[float, float]:
    """(CFL signal, max wavespeed) over the interior (timeint.py:115-131)."""
    G = prob.geom()
    out = np.zeros(2)
    where = ctypes.c_int64(-1)
    rc = lib().or_max_signal(ctypes.byref(G), _p(u), 1 if cfl_mode == "sum" else 0, _p(out),
                             ctypes.byref(where))
    if rc:
        raise OracleStateError(rc, where.value)
    return float(out[0]), float(out[1])


def enstrophy(u: np.ndarray, prob: Problem) -> float:
    """Mean of 0.5 |curl(m/rho)|^2 over the interior (ghosts refilled first)."""
    fill_ghosts(u, prob)
    G = prob.geom()
    return float(lib().or_enstrophy(ctypes.byref(G), _p(u))) / (prob.n[0] * prob.n[1] * prob.n[2])


def advance(u: np.ndarray, prob: Problem, steps: int, cfl: float | None = 0.4,
            dt: float | None = None, scheme: str = "rk4") -> np.ndarray:
    """``steps`` steps in place; returns the dt sequence (timeint.py:199-258)."""
    G = prob.geom()
    dts = np.zeros(max(steps, 1))
    where = ctypes.c_int64(-1)
    rc = lib().or_advance(ctypes.byref(G), _p(u), 3 if scheme == "rk3" else 4,
                          float(cfl or 0.0), float(dt or 0.0), int(steps), _p(dts),
                          ctypes.byref(where))
    if rc:
        # steps 1..k-1 completed; step k stored its dt unless its CFL reduction failed (rc >= 100)
        k = int(np.count_nonzero(dts)) + (1 if rc >= 100 else 0)
        raise OracleStateError(rc % 10, where.value, stage=(rc // 10) % 10, step=k)
    return dts[:steps]


def interior(u: np.ndarray, prob: Problem) -> np.ndarray:
    g = prob.g
    v = u.reshape((5,) + prob.shape)
    return v[:, g:g + prob.n[2], g:g + prob.n[1], g:g + prob.n[0]]


def from_interior(body: np.ndarray, prob: Problem) -> np.ndarray:
    """Ghosted flat buffer (ghosts filled) from a (5, nz, ny, nx) interior."""
    u = np.zeros(5 * prob.npts)
    interior(u, prob)[...] = body
    return fill_ghosts(u, prob)


def bench_weights(values: np.ndarray, nx: int, ny: int, nz: int, pad: int = 2,
                  eps: float = 1e-6, power: int = 2) -> np.ndarray:
    """Point-major weights of the layout study (kernels.py:243-291) from the
    canonical (points, 5) values: out[3 * (5 p + v) + 0..2] for the active
    points, zero elsewhere.  numpy evaluates every binary op in IEEE double
    without contraction, in the association order written below -- the same
    as the numba kernel (pinned by tests/golden/bench_weights.npz)."""
    px = nx + 2 * pad
    npts = px * ny * nz
    out = np.zeros((npts, 5, 3))
    p = (np.arange(nz)[:, None, None] * ny + np.arange(ny)[None, :, None]) * px + pad + \
        np.arange(nx)[None, None, :]
    p = p.reshape(-1)
    for v in range(5):
        f0, f1, f2, f3, f4 = (values[p + s, v] for s in (-2, -1, 0, 1, 2))
        t1 = (f0 - 2.0 * f1) + f2
        s1 = (f0 - 4.0 * f1) + 3.0 * f2
        b1 = (13.0 / 12.0) * (t1 * t1) + 0.25 * (s1 * s1)
        t2 = (f1 - 2.0 * f2) + f3
        s2 = f1 - f3
        b2 = (13.0 / 12.0) * (t2 * t2) + 0.25 * (s2 * s2)
        t3 = (f2 - 2.0 * f3) + f4
        s3 = (3.0 * f2 - 4.0 * f3) + f4
        b3 = (13.0 / 12.0) * (t3 * t3) + 0.25 * (s3 * s3)
        d1, d2, d3 = eps + b1, eps + b2, eps + b3
        e1, e2, e3 = d1, d2, d3
        for _ in range(power - 1):
            e1, e2, e3 = e1 * d1, e2 * d2, e3 * d3
        a1, a2, a3 = 0.1 / e1, 0.6 / e2, 0.3 / e3
        asum = (a1 + a2) + a3
        out[p, v, 0] = a1 / asum
        out[p, v, 1] = a2 / asum
        out[p, v, 2] = a3 / asum
    return out.reshape(-1)
