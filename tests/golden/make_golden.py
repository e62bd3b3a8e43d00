"""Generate the golden fixtures by running the reference package itself.

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden.py

Everything written here comes from the UNMODIFIED reference
(pkg/src/hitdns) on its public API; the fixtures pin both the C oracle
(tests/test_oracle_golden.py) and, through it, the CUDA product.

Fixtures (tests/golden/):
  kernels.npz   per-kernel vectors: hyper_sweep per dim (kernels.py:69) on a
                rough random state of a non-cubic grid, central_diff4
                (kernels.py:208), hyperbolic_rhs / parabolic_rhs / rhs
                (upwind.py:163, viscous.py:54, timeint.py:141) incl. the
                entropy-fix (delta>0) and power=3 variants
  traj16.npz    16^3 HIT IC, 10 RK4 steps at CFL 0.4, mu=0.006: per-step
                dt, totals, max wavespeed and the final interior state;
                3 RK3 steps for the TVD-RK3 stepper
  bench_weights.npz  layout-study weight kernel (kernels.py:292-329 via
                bench.py:102 run_case): outputs of the 4 layout x traversal
                cases on a ragged (9, 5, 3) grid (all bitwise equal) and the
                canonical values of bench.make_bench_values
  traj32.json   config 1 (32^3, RK4, CFL 0.4, mu=0.006, 10 steps): IC and
                final SHA-256, per-variable L2, dts, KE per step,
                enstrophy per step (the north star's diagnostic, built from the
                reference's decode_primitives + central_derivative_4)
  viscous_limit.json  16^3 HIT, RK4, CFL 0.4 at mu = 0.3 (dt beyond the viscous
                operator's RK4 limit): the StepError step / stage / kind the
                reference raises; at mu = 0.2: 60 steps complete, final t and dts
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = os.environ.get("HITDNS_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nb")

import hitdns as hd  # noqa: E402
from hitdns import kernels  # noqa: E402
from hitdns.upwind import _flux_components  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
MU = 0.006


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def rough_state(n, length, seed=7):
    """Random positive primitives per cell: exercises nonlinear WENO weights."""
    rng = np.random.default_rng(seed)
    spec = hd.GridSpec(n=n, length=length)
    shape = spec.interior_shape
    rho = 0.6 + 0.8 * rng.random(shape)
    u = 0.5 * rng.standard_normal(shape)
    v = 0.5 * rng.standard_normal(shape)
    w = 0.5 * rng.standard_normal(shape)
    p = 0.7 + 0.6 * rng.random(shape)
    fs = hd.FieldSet.zeros(spec)
    it = fs.interior()
    it[0] = rho
    it[1] = rho * u
    it[2] = rho * v
    it[3] = rho * w
    it[4] = p / 0.4 + 0.5 * rho * (u * u + v * v + w * w)
    hd.fill_ghosts_periodic(fs)
    return fs


def kernel_vectors():
    out = {}
    n = (12, 10, 8)
    length = (2.0, 1.5, 1.0)
    fs = rough_state(n, length)
    spec = fs.spec
    out["rough_n"] = np.array(n)
    out["rough_length"] = np.array(length)
    out["rough_u"] = fs.data.copy()
    gas = hd.GasModel()
    # per-dimension hyper_sweep, as hyperbolic_rhs drives it (upwind.py:186-212)
    view = fs.component_view()
    prims = hd.decode_primitives(fs, gas.gamma)
    gz, gy, gx = spec.shape
    sx, sy, sz = 1, gx, gx * gy
    g = spec.ghost_width
    base0 = g * sz + g * sy + g * sx
    nx, ny, nz = spec.n
    geom = ((sx, sz, sy, nx, nz, ny), (sy, sz, sx, ny, nz, nx), (sz, sy, sx, nz, ny, nx))
    for dim in range(3):
        flux = _flux_components(view, prims, dim).reshape(-1)
        inc = np.zeros_like(fs.data)
        sd, sa, sb, nd, na, nb = geom[dim]
        kernels.hyper_sweep(fs.data, flux, inc, spec.total_points, base0, sd, sa, sb, nd, nb, 0,
                            na, dim, 1.0 / spec.spacing[dim], gas.gamma, 1e-6, 2, 0.0)
        out[f"sweep{dim}_flux"] = flux
        out[f"sweep{dim}_inc"] = inc
    out["hyper"] = hd.hyperbolic_rhs(fs, gas).data
    out["hyper_delta"] = hd.hyperbolic_rhs(fs, gas, delta=0.3).data
    out["hyper_p3"] = hd.hyperbolic_rhs(fs, gas, params=hd.WenoParams(epsilon=1e-5, power=3)).data
    out["parab"] = hd.parabolic_rhs(fs, hd.GasModel(mu=MU)).data
    out["rhs"] = hd.make_rhs(hd.GasModel(mu=MU))(fs.copy()).data
    # central_diff4 on one ghosted scalar (variable 4), each dimension
    e = view[4]
    for d in range(3):
        out[f"cd4_{d}"] = hd.central_derivative_4(e, d, spec.spacing[d], g)
    # rhs on a fresh (ghost-unfilled) state: the rhs must fill ghosts itself
    raw = fs.copy()
    hd.FieldSet  # noqa: B018
    rv = raw.component_view()
    rv[:, :g] = 0.0
    out["rhs_unfilled_u"] = raw.data.copy()
    out["rhs_unfilled"] = hd.make_rhs(hd.GasModel(mu=MU))(raw).data
    np.savez_compressed(os.path.join(OUT, "kernels.npz"), **out)


def trajectory16():
    spec = hd.GridSpec((16, 16, 16))
    ic = hd.make_initial_condition(spec, hd.HitParams())
    gas = hd.GasModel(mu=MU)
    res = hd.advance(ic.copy(), gas, hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=10))
    rec = res.records
    rk3 = hd.advance(ic.copy(), gas, hd.TimeParams(scheme="rk3", cfl=0.4, max_steps=3))
    np.savez_compressed(
        os.path.join(OUT, "traj16.npz"),
        ic=ic.interior().copy(),
        final=res.fields.interior().copy(),
        t=np.array(res.t),
        dt=np.array([r.dt for r in rec]),
        mass=np.array([r.mass for r in rec]),
        momentum=np.array([r.momentum for r in rec]),
        energy=np.array([r.energy for r in rec]),
        max_wavespeed=np.array([r.max_wavespeed for r in rec]),
        rk3_final=rk3.fields.interior().copy(),
        rk3_dt=np.array([r.dt for r in rk3.records]),
    )


def enstrophy(fields) -> float:
    """0.5 <|curl v|^2> with the reference's own operators: velocities from
    decode_primitives (physics.py:240-255), each derivative central_derivative_4
    (viscous.py:23-51)."""
    fs = fields.copy()
    hd.fill_ghosts_periodic(fs)
    _, u, v, w, _ = hd.decode_primitives(fs, 1.4)
    h, g = fs.spec.spacing, fs.spec.ghost_width

    def D(a, d):
        return hd.central_derivative_4(a, d, h[d], g)

    wx, wy, wz = D(w, 1) - D(v, 2), D(u, 2) - D(w, 0), D(v, 0) - D(u, 1)
    return float(np.mean(0.5 * ((wx * wx + wy * wy) + wz * wz)))


def trajectory32():
    spec = hd.GridSpec((32, 32, 32))
    ic = hd.make_initial_condition(spec, hd.HitParams())
    gas = hd.GasModel(mu=MU)
    fields = ic.copy()
    t = 0.0
    dts, kes, ens = [], [], [enstrophy(ic)]
    it = ic.interior()
    kes.append(hd.compute_spectrum(it[1] / it[0], it[2] / it[0], it[3] / it[0]).total())
    for _ in range(10):
        res = hd.advance(fields, gas, hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=1), t0=t)
        fields, t = res.fields, res.t
        dts.append(res.records[0].dt)
        it = fields.interior()
        kes.append(hd.compute_spectrum(it[1] / it[0], it[2] / it[0], it[3] / it[0]).total())
        ens.append(enstrophy(fields))
    final = fields.interior()
    doc = {
        "config": "32^3 HIT IC (HitParams defaults, seed 2024), GasModel(mu=0.006), RK4, CFL 0.4, 10 steps",
        "numpy": np.__version__,
        "ic_sha256": sha(ic.interior()),
        "final_sha256": sha(final),
        "t": t,
        "dt": dts,
        "ke": kes,
        "enstrophy": ens,
        "l2": [float(np.sqrt(np.sum(final[v] ** 2))) for v in range(5)],
        "mass": res.records[0].mass,
        "energy": res.records[0].energy,
    }
    with open(os.path.join(OUT, "traj32.json"), "w") as fh:
        json.dump(doc, fh, indent=1)
    print(json.dumps(doc, indent=1))


def viscous_limit():
    n = 16
    spec = hd.GridSpec((n, n, n))
    ic = hd.make_initial_condition(spec, hd.HitParams())
    doc = {"n": n, "cfl": 0.4, "scheme": "rk4", "max_steps": 60}
    try:
        hd.advance(ic, hd.GasModel(mu=0.3), hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=60))
        raise SystemExit("expected StepError at mu = 0.3")
    except hd.StepError as e:
        doc["unstable"] = {"mu": 0.3, "step": int(e.step), "stage": int(e.stage),
                           "message": str(e)}
    r = hd.advance(ic, hd.GasModel(mu=0.2), hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=60))
    doc["stable"] = {"mu": 0.2, "steps": len(r.records), "t": r.t,
                     "dts": [rec.dt for rec in r.records]}
    with open(os.path.join(OUT, "viscous_limit.json"), "w") as fh:
        json.dump(doc, fh, indent=1)


def bench_weights():
    from hitdns import bench

    shape = (9, 5, 3)
    out = {"shape": np.array(shape), "values": bench.make_bench_values(shape)}
    for layout in (hd.Layout.INTERLEAVED, hd.Layout.COMPONENT_CONTIGUOUS):
        for trav in ("lex", "tiled"):
            rec, w = bench.run_case(shape, layout, trav, repeats=1)
            out[f"out_{int(layout)}_{trav}"] = w
            out[f"wasted_{int(layout)}_{trav}"] = np.array(rec.wasted_lanes)
    np.savez_compressed(os.path.join(OUT, "bench_weights.npz"), **out)


if __name__ == "__main__":
    import sys as _sys

    if _sys.argv[1:] == ["bench_weights"]:
        bench_weights()
        raise SystemExit(0)
    if _sys.argv[1:] == ["trajectory32"]:
        trajectory32()
        raise SystemExit(0)
    if _sys.argv[1:] == ["viscous_limit"]:
        viscous_limit()
        raise SystemExit(0)
    bench_weights()
    kernel_vectors()
    trajectory16()
    trajectory32()
    viscous_limit()
