"""CUDA path (libhd.so through the package API) against the oracle and the
reference's golden vectors.

Tolerances:
* exact mode -- bitwise (np.array_equal) against vectors produced by the
  reference itself: the kernels follow the reference operation order with
  no FMA contraction;
* fast mode -- the north-star bar, relative L2 <= 1e-10 per conserved
  variable after N steps (BASELINE.json), and per-kernel max error
  <= 1e-12 relative to the field scale.
"""

import hashlib

import numpy as np
import pytest
import torch

from conftest import rough_problem

pytestmark = pytest.mark.gpu

FAST_KERNEL_TOL = 1e-12
TRAJ_TOL = 1e-10


@pytest.fixture(scope="module")
def hd():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2211_16718_b200 as hd

    hd._lib.load(require_cuda=True)
    return hd


def _spec(hd, P):
    return hd.GridSpec(P.n, P.length)


def _fs(hd, P, flat):
    return hd.FieldSet(_spec(hd, P), hd.Layout.COMPONENT_CONTIGUOUS, torch.from_numpy(flat.copy()).cuda())


def _rel_l2(a, b):
    a = a.reshape(5, -1)
    b = b.reshape(5, -1)
    return np.sqrt(np.sum((a - b) ** 2, axis=1)) / np.maximum(np.sqrt(np.sum(b ** 2, axis=1)), 1e-300)


def _close(a, b, tol):
    scale = max(np.max(np.abs(b)), 1e-300)
    return np.max(np.abs(a - b)) <= tol * scale


@pytest.mark.parametrize("mode", ["exact", "fast"])
@pytest.mark.parametrize("dim", [0, 1, 2])
def test_hyper_sweep(hd, kernels_golden, mode, dim):
    K = kernels_golden
    P = rough_problem(K)
    fs = _fs(hd, P, K["rough_u"])
    inc = fs.like()
    hd.hyper_sweep(fs, dim, inc, mode=mode)
    got = inc.numpy()
    want = K[f"sweep{dim}_inc"]
    if mode == "exact":
        assert np.array_equal(got, want)
    else:
        assert _close(got, want, FAST_KERNEL_TOL)


@pytest.mark.parametrize("mode", ["exact", "fast"])
@pytest.mark.parametrize("name,kw", [
    ("hyper", {}),
    ("hyper_delta", {"delta": 0.3}),
    ("hyper_p3", {"params": "p3"}),
])
def test_hyperbolic_rhs(hd, kernels_golden, mode, name, kw):
    K = kernels_golden
    P = rough_problem(K)
    fs = _fs(hd, P, K["rough_u"])
    params = hd.WenoParams(epsilon=1e-5, power=3) if kw.get("params") == "p3" else hd.DEFAULT_PARAMS
    out = hd.hyperbolic_rhs(fs, hd.GasModel(), params, kw.get("delta", 0.0), mode=mode).numpy()
    if mode == "exact":
        assert np.array_equal(out, K[name])
    else:
        assert _close(out, K[name], FAST_KERNEL_TOL)


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_make_rhs(hd, kernels_golden, mode):
    K = kernels_golden
    P = rough_problem(K)
    rhs = hd.make_rhs(hd.GasModel(mu=0.006), mode=mode)
    for src, name in (("rough_u", "rhs"), ("rhs_unfilled_u", "rhs_unfilled")):
        out = rhs(_fs(hd, P, K[src])).numpy()
        if mode == "exact":
            assert np.array_equal(out, K[name]), name
        else:
            assert _close(out, K[name], FAST_KERNEL_TOL), name


@pytest.mark.parametrize("dim", [0, 1, 2])
def test_central_derivative_4(hd, kernels_golden, dim):
    K = kernels_golden
    P = rough_problem(K)
    e = torch.from_numpy(K["rough_u"].reshape((5,) + P.shape)[4].copy()).cuda()
    out = hd.central_derivative_4(e, dim, P.length[dim] / P.n[dim], 3)
    assert np.array_equal(out.cpu().numpy(), K[f"cd4_{dim}"])


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_rk4_trajectory16(hd, oracle, traj16_golden, mode):
    T = traj16_golden
    P = oracle.Problem(n=(16, 16, 16), mu=0.006)
    fs = _fs(hd, P, oracle.from_interior(T["ic"], P))
    res = hd.advance(fs, hd.GasModel(mu=0.006), hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=10),
                     mode=mode)
    got = res.fields.interior().cpu().numpy()
    dts = np.array([r.dt for r in res.records])
    if mode == "exact":
        assert np.array_equal(dts, T["dt"])
        assert np.array_equal(got, T["final"])
        assert res.t == float(T["t"])
    else:
        assert np.max(np.abs(dts - T["dt"]) / T["dt"]) < 1e-12
        assert np.all(_rel_l2(got, T["final"]) <= TRAJ_TOL)
    mass = np.array([r.mass for r in res.records])
    energy = np.array([r.energy for r in res.records])
    assert np.allclose(mass, T["mass"], rtol=1e-13, atol=0)
    assert np.allclose(energy, T["energy"], rtol=1e-13, atol=0)
    assert np.allclose([r.max_wavespeed for r in res.records], T["max_wavespeed"], rtol=1e-12)


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_rk3_trajectory16(hd, oracle, traj16_golden, mode):
    T = traj16_golden
    P = oracle.Problem(n=(16, 16, 16), mu=0.006)
    fs = _fs(hd, P, oracle.from_interior(T["ic"], P))
    res = hd.advance(fs, hd.GasModel(mu=0.006), hd.TimeParams(scheme="rk3", cfl=0.4, max_steps=3),
                     mode=mode)
    got = res.fields.interior().cpu().numpy()
    if mode == "exact":
        assert np.array_equal(got, T["rk3_final"])
    else:
        assert np.all(_rel_l2(got, T["rk3_final"]) <= TRAJ_TOL)


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_config1_trajectory(hd, traj32_golden, mode):
    """Config 1: 32^3 HIT IC, RK4, CFL 0.4, mu 0.006, 10 steps,
    with the reference's kinetic-energy decay curve."""
    G = traj32_golden
    spec = hd.GridSpec((32, 32, 32))
    ic = hd.make_initial_condition(spec, hd.HitParams(), backend="numpy")
    assert hashlib.sha256(ic.interior().cpu().numpy().tobytes()).hexdigest() == G["ic_sha256"]
    res = hd.advance(ic, hd.GasModel(mu=0.006), hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=10),
                     mode=mode)
    fin = res.fields.interior().cpu().numpy()
    l2 = np.sqrt(np.sum(fin.reshape(5, -1) ** 2, axis=1))
    ke = [r.kinetic_energy for r in res.records]
    if mode == "exact":
        assert hashlib.sha256(fin.tobytes()).hexdigest() == G["final_sha256"]
        assert [r.dt for r in res.records] == G["dt"]
        assert res.t == G["t"]
    assert np.all(np.abs(l2 - np.array(G["l2"])) / np.array(G["l2"]) <= TRAJ_TOL)
    assert np.allclose(ke, G["ke"][1:], rtol=1e-11, atol=0)
    # enstrophy per step (north star; golden from the reference's operators): the
    # previous step's result folded into each step's first flux kernel, the last
    # one a separate pass
    ens = [r.enstrophy for r in res.records]
    assert np.allclose(ens, G["enstrophy"][1:], rtol=1e-11, atol=0)
    assert abs(hd.enstrophy(ic) - G["enstrophy"][0]) <= 1e-12 * G["enstrophy"][0]


@pytest.mark.parametrize("mu", [0.006, 0.0])
def test_enstrophy_paths_agree(hd, mu):
    """Folded into the stage-0 flux kernel (eager march), the stand-alone pass
    (observer march, inviscid runs, final state) and the public function agree."""
    spec = hd.GridSpec((32, 32, 32))
    ic = hd.make_initial_condition(spec, hd.HitParams(), backend="numpy")
    tp = hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=4)
    gas = hd.GasModel(mu=mu)
    a = hd.advance(ic, gas, tp)
    seen = []
    b = hd.advance(ic, gas, tp, observer=seen.append)
    ea = np.array([r.enstrophy for r in a.records])
    eb = np.array([r.enstrophy for r in b.records])
    assert np.all(np.isfinite(ea)) and len(seen) == 4
    assert np.allclose(ea, eb, rtol=1e-13, atol=0)
    assert np.isclose(hd.enstrophy(a.fields), ea[-1], rtol=1e-13, atol=0)


def test_fast_vs_exact_32(hd):
    spec = hd.GridSpec((32, 32, 32))
    ic = hd.make_initial_condition(spec, hd.HitParams(), backend="numpy")
    tp = hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=20)
    a = hd.advance(ic, hd.GasModel(mu=0.006), tp, mode="exact").fields.interior().cpu().numpy()
    b = hd.advance(ic, hd.GasModel(mu=0.006), tp, mode="fast").fields.interior().cpu().numpy()
    assert np.all(_rel_l2(b, a) <= TRAJ_TOL)


def test_step_error_reports_stage(hd):
    """Negative energy -> StepError with step and stage (test_timeint.py:161-171)."""
    spec = hd.GridSpec((8, 8, 8))
    fs = hd.FieldSet.zeros(spec)
    it = fs.interior()
    it[0] = 1.0
    it[4] = 2.5
    it[4, 2, 3, 4] = -1.0
    # CFL sizing decodes the state first: compute_dt raises InvalidStateError (timeint.py:235)
    with pytest.raises(hd.InvalidStateError) as ei:
        hd.advance(fs, hd.GasModel(), hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=2))
    assert not isinstance(ei.value, hd.StepError)
    # fixed dt: the first RHS decode fails -> StepError(step 1, stage 0) (timeint.py:161-165, 238-241)
    with pytest.raises(hd.StepError) as ei:
        hd.advance(fs, hd.GasModel(), hd.TimeParams(scheme="rk4", dt=0.01, max_steps=2))
    assert ei.value.step == 1 and ei.value.stage == 0
    # a valid state with an absurd fixed dt: the stage-1 input u + (dt/2) k1 has
    # negative density, so the second RHS evaluation fails -> StepError(step 1, stage 1)
    fs2 = hd.FieldSet.zeros(spec)
    x = torch.arange(8, dtype=torch.float64, device="cuda") * (2 * np.pi / 8)
    w = 0.9 * torch.sin(x)[:, None, None]  # z velocity varying along z
    fs2.interior()[0] = 1.0
    fs2.interior()[3] = w
    fs2.interior()[4] = 2.5 + 0.5 * w * w
    with pytest.raises(hd.StepError) as ei:
        hd.advance(fs2, hd.GasModel(), hd.TimeParams(scheme="rk4", dt=50.0, max_steps=3))
    assert ei.value.step == 1 and ei.value.stage == 1


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_viscous_time_step_limit_fails_like_the_reference(hd, viscous_limit_golden, mode):
    """The reference's dt is convective only (timeint.py:122-138); when the
    viscosity makes the fourth-order viscous operator RK4-unstable at that dt
    (dt > ~42 h^2 at mu = 0.006, i.e. n >~ 900; here n = 16 with mu = 0.3) the
    march grows the highest modes until a pressure goes negative.  The GPU march
    must stop at the step and stage the reference stops at
    (tests/golden/viscous_limit.json; exact mode: the same trajectory, bit for
    bit; fast mode: within one step), and the stable viscosity must run through
    (exact mode: the reference's dt sequence)."""
    G = viscous_limit_golden
    n = G["n"]
    spec = hd.GridSpec((n,) * 3)
    ic = hd.make_initial_condition(spec, hd.HitParams(), backend="numpy")
    bad, ok = G["unstable"], G["stable"]
    with pytest.raises(hd.StepError) as ge:
        hd.advance(ic, hd.GasModel(mu=bad["mu"]),
                   hd.TimeParams(scheme="rk4", cfl=G["cfl"], max_steps=G["max_steps"]), mode=mode)
    assert ge.value.stage == bad["stage"]
    assert "pressure" in str(ge.value)
    if mode == "exact":
        assert ge.value.step == bad["step"]
        # the same array index as the reference: the first offending cell in C order
        # over the filled ghosted box -- here a ghost image (z = 0)
        inner = ge.value
        while not hasattr(inner, "where"):
            inner = inner.__cause__
        assert tuple(int(c) for c in inner.where) == (0, 8, 9)
        assert f"at array index {inner.where}" in str(ge.value)
    else:
        assert abs(ge.value.step - bad["step"]) <= 1
    res = hd.advance(ic, hd.GasModel(mu=ok["mu"]),
                     hd.TimeParams(scheme="rk4", cfl=G["cfl"], max_steps=G["max_steps"]), mode=mode)
    assert res.steps == G["max_steps"]
    if mode == "exact":
        assert [r.dt for r in res.records] == ok["dts"]


def test_uniform_flow_zero_rhs(hd):
    n = 12
    spec = hd.GridSpec((n, n, n))
    fs = hd.FieldSet.zeros(spec)
    it = fs.interior()
    rho, u, p = 1.1, 0.4, 0.9
    it[0] = rho
    it[1] = rho * u
    it[2] = rho * 0.2 * u
    it[3] = -rho * 0.1 * u
    it[4] = p / 0.4 + 0.5 * rho * (u * u * (1 + 0.04 + 0.01))
    hd.fill_ghosts_periodic(fs)
    for mode in ("exact", "fast"):
        out = hd.hyperbolic_rhs(fs, hd.GasModel(), mode=mode)
        assert out.interior().abs().max().item() < 1e-13


def test_fixed_dt_lands_on_t_final(hd):
    spec = hd.GridSpec((16, 16, 16))
    ic = hd.make_initial_condition(spec, hd.HitParams(), backend="numpy")
    seen = []
    res = hd.advance(ic, hd.GasModel(mu=0.006), hd.TimeParams(scheme="rk4", dt=0.03, t_final=0.1),
                     observer=seen.append)
    assert res.steps == 4 and len(seen) == 4
    assert abs(res.t - 0.1) < 1e-15
    assert abs(res.records[-1].dt - (0.1 - 0.09)) < 1e-15


def test_inviscid_conservation(hd):
    """Acceptance analogue (test_acceptance.py:315-341) on 32^3, 40 RK4 steps."""
    spec = hd.GridSpec((32, 32, 32))
    ic = hd.make_initial_condition(spec, hd.HitParams(), backend="numpy")
    m0, mom0, e0 = hd.conserved_totals(ic)
    res = hd.advance(ic, hd.GasModel(), hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=40))
    m1, mom1, e1 = hd.conserved_totals(res.fields)
    assert abs(m1 - m0) / abs(m0) < 1e-11
    assert abs(e1 - e0) / abs(e0) < 1e-11
    assert max(abs(a - b) for a, b in zip(mom0, mom1)) < 1e-11


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_x_sweep_staged_matches_unstaged(hd, oracle, monkeypatch, mode):
    """The shared-memory staged x sweep (n_y % 32 == 0) is bitwise the plain x sweep,
    and in exact mode bitwise the oracle (kernels.py:68-204 on x lines)."""
    rng = np.random.default_rng(11)
    P = oracle.Problem(n=(24, 64, 6), length=(1.0, 2.0, 0.5))
    body = np.empty((5,) + (6, 64, 24))
    rho = 0.6 + 0.8 * rng.random(body.shape[1:])
    vel = 0.5 * rng.standard_normal((3,) + body.shape[1:])
    p = 0.7 + 0.6 * rng.random(body.shape[1:])
    body[0] = rho
    body[1:4] = rho * vel
    body[4] = p / 0.4 + 0.5 * rho * (vel ** 2).sum(0)
    u = oracle.from_interior(body, P)
    fs = _fs(hd, P, u)
    outs = []
    for staged in (1, 0):
        hd.get_plan(fs.spec, hd.GasModel(), mode=mode).set_option(hd._lib.HD_OPT_X_STAGED, staged)
        inc = fs.like()
        inc.data.fill_(0.25)
        hd.hyper_sweep(fs, 0, inc, mode=mode)
        outs.append(inc.numpy())
    hd.get_plan(fs.spec, hd.GasModel(), mode=mode).set_option(hd._lib.HD_OPT_X_STAGED, 1)
    if mode == "exact":
        assert np.array_equal(outs[0], outs[1])
    else:  # different kernels may contract FMAs differently
        assert _close(outs[1], outs[0], 1e-13)
    if mode == "exact":
        gz, gy, gx = P.shape
        g = 3
        flux = np.empty_like(u)
        prim = u.reshape(5, -1)
        inv = 1.0 / prim[0]
        vx = prim[1] * inv
        pp = (1.4 - 1.0) * (prim[4] - 0.5 * prim[0] * ((vx * vx + (prim[2] * inv) ** 2) + (prim[3] * inv) ** 2))
        f = flux.reshape(5, -1)
        f[0] = prim[1]
        f[1] = prim[1] * vx + pp
        f[2] = prim[2] * vx
        f[3] = prim[3] * vx
        f[4] = (prim[4] + pp) * vx
        want = np.full_like(u, 0.25)
        want.reshape(5, *P.shape)[:, :g] = 0.25
        ref = np.zeros_like(u)
        ref[:] = 0.25
        oracle.hyper_sweep(u, flux, ref, P.npts, g * gx * gy + g * gx + g, 1, gx * gy, gx, 24, 64,
                           0, 6, 0, 1.0 / (1.0 / 24), 1.4, 1e-6, 2, 0.0)
        inner = oracle.interior
        assert np.array_equal(inner(outs[0], P), inner(ref, P))


def _smooth_state(P):
    """A smooth, non-trivial periodic state on P's grid (every kernel path exercised)."""
    nz, ny, nx = P.n[2], P.n[1], P.n[0]
    z, y, x = np.meshgrid(*(np.arange(m) * (2 * np.pi / m) for m in (nz, ny, nx)), indexing="ij")
    rho = 1.0 + 0.2 * np.sin(x) * np.cos(2 * y) + 0.1 * np.cos(z)
    u = 0.3 * np.sin(y + z)
    v = 0.25 * np.cos(x - z)
    w = 0.2 * np.sin(2 * x + y)
    p = 0.8 + 0.1 * np.cos(x + y + z)
    body = np.stack([rho, rho * u, rho * v, rho * w,
                     p / 0.4 + 0.5 * rho * (u * u + v * v + w * w)])
    return body


@pytest.mark.parametrize("mode", ["exact", "fast"])
@pytest.mark.parametrize("n", [(32, 24, 20), (40, 32, 12), (24, 16, 40)])
def test_ragged_grids_match_oracle(hd, oracle, mode, n):
    """Grids off the fast paths' tile multiples (staged x sweep needs n_y % 32,
    the z-marching flux kernel n_x % 32 and n_y % 8) take the general kernels;
    every combination must still match the oracle: 4 RK4 steps, viscous."""
    P = oracle.Problem(n=n, length=(2 * np.pi, 1.5 * np.pi, np.pi), mu=0.01)
    u = oracle.from_interior(_smooth_state(P), P)
    fs = _fs(hd, P, u)
    want = u.copy()
    dts = oracle.advance(want, P, 4, cfl=0.4)
    res = hd.advance(fs, hd.GasModel(mu=0.01), hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=4),
                     mode=mode)
    got = res.fields.interior().cpu().numpy()
    ref = oracle.interior(want, P)
    if mode == "exact":
        assert np.array_equal(got, ref)
        assert np.array_equal(np.array([r.dt for r in res.records]), dts)
    else:
        assert np.all(_rel_l2(got, ref) <= TRAJ_TOL)
