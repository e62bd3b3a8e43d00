"""The reference's acceptance criteria (pkg/tests/test_acceptance.py) run on the CUDA path.

* fifth-order advected density wave, 32 -> 64 -> 128 (:119-146): order >= 4.5
* fourth-order viscous operators on a shear profile, 32 -> 64 (:149-174): order >= 3.5
* results independent of how lines are split into segments -- the analogue
  of the reference's worker-count invariance (pkg/tests/test_upwind.py:107-111)
"""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

GAMMA = 1.4


@pytest.fixture(scope="module")
def hd():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2211_16718_b200 as hd

    hd._lib.load(require_cuda=True)
    return hd


def _coords(n):
    c = torch.arange(n, dtype=torch.float64, device="cuda") * (2 * math.pi / n)
    return torch.meshgrid(c, c, c, indexing="ij")  # z, y, x


def _from_prims(hd, spec, rho, u, v, w, p):
    fs = hd.FieldSet.zeros(spec)
    it = fs.interior()
    it[0] = rho
    it[1] = rho * u
    it[2] = rho * v
    it[3] = rho * w
    it[4] = p / (GAMMA - 1.0) + 0.5 * rho * (u * u + v * v + w * w)
    hd.fill_ghosts_periodic(fs)
    return fs


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_fifth_order_advected_density(hd, mode):
    wind, amp, p0 = 0.7, 0.3, 1.0
    errs = []
    for n in (32, 64, 128):
        spec = hd.GridSpec((n, n, n))
        z, y, x = _coords(n)
        rho = 1.0 + amp * torch.sin(x)
        one = torch.ones_like(rho)
        fs = _from_prims(hd, spec, rho, wind * one, 0 * one, 0 * one, p0 * one)
        inc = hd.hyperbolic_rhs(fs, hd.GasModel(), mode=mode).interior()
        drho = amp * torch.cos(x)
        want = torch.zeros_like(inc)
        want[0] = -wind * drho
        want[1] = -wind * wind * drho
        want[4] = -0.5 * wind ** 3 * drho
        errs.append((inc - want).abs().max().item())
    o1, o2 = math.log2(errs[0] / errs[1]), math.log2(errs[1] / errs[2])
    assert o1 >= 4.5 and o2 >= 4.5, (o1, o2)


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_fourth_order_viscous_on_shear(hd, mode):
    mu = 0.01
    errs_d, errs_m, errs_e = [], [], []
    for n in (32, 64):
        spec = hd.GridSpec((n, n, n))
        z, y, x = _coords(n)
        g = spec.ghost_width
        buf = torch.zeros(spec.shape, dtype=torch.float64, device="cuda")
        buf[g:-g, g:-g, g:-g] = torch.sin(y)
        hd.fill_ghosts_array(buf, spec.n, g)
        got = hd.central_derivative_4(buf, 1, spec.spacing[1])
        errs_d.append((got - torch.cos(y)).abs().max().item())
        zero = torch.zeros_like(y)
        fs = _from_prims(hd, spec, torch.ones_like(y), torch.sin(y), zero, zero,
                         torch.full_like(y, 1.0 / GAMMA))
        inc = hd.parabolic_rhs(fs, hd.GasModel(mu=mu), mode=mode).interior()
        errs_m.append((inc[1] + mu * torch.sin(y)).abs().max().item())
        errs_e.append((inc[4] - mu * torch.cos(2.0 * y)).abs().max().item())
    for e in (errs_d, errs_m, errs_e):
        assert math.log2(e[0] / e[1]) >= 3.5


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_segment_split_invariance(hd, monkeypatch, mode):
    """One thread per line, or the line cut into 4 or 7 segments: every
    interface is evaluated from the same window, so the step is bitwise equal."""
    spec = hd.GridSpec((32, 64, 56))
    rng = np.random.default_rng(5)
    shape = spec.interior_shape
    rho = torch.from_numpy(0.8 + 0.4 * rng.random(shape)).cuda()
    vel = [torch.from_numpy(0.3 * rng.standard_normal(shape)).cuda() for _ in range(3)]
    p = torch.from_numpy(0.8 + 0.4 * rng.random(shape)).cuda()
    fs = _from_prims(hd, spec, rho, *vel, p)
    outs = []
    for segs in (1, 4, 7):
        hd.release_plans()
        hd.get_plan(spec, hd.GasModel(mu=0.01), mode=mode).set_option(hd._lib.HD_OPT_SEGMENTS, segs)
        res = hd.advance(fs, hd.GasModel(mu=0.01), hd.TimeParams(scheme="rk4", cfl=0.3, max_steps=2),
                         mode=mode)
        outs.append(res.fields.interior().cpu().numpy())
    hd.release_plans()
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


def test_torch_ic_is_reproducible(hd):
    """The GPU synthesis (used at 512^3, one copy per rank) is bit-for-bit
    reproducible: every rank of a decomposed run starts from the same state."""
    spec = hd.GridSpec((64, 64, 64))
    a = hd.make_initial_condition(spec, hd.HitParams(), backend="torch").data
    b = hd.make_initial_condition(spec, hd.HitParams(), backend="torch").data
    assert torch.equal(a, b)


GAMMA_HIT = 1.4


def _vel(fields):
    it = fields.interior()
    return it[1] / it[0], it[2] / it[0], it[3] / it[0]


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_inviscid_hundred_step_conservation(hd, mode):
    """pkg/tests/test_acceptance.py:315-341 as written: 64^3, mu = 0, the default
    TimeParams scheme (RK3), CFL 0.4, 100 steps; drifts < 1e-11."""
    params = hd.HitParams()
    spec = hd.GridSpec((64, 64, 64))
    fields = hd.make_initial_condition(spec, params, GAMMA_HIT, backend="numpy")
    mass0, mom0, energy0 = hd.conserved_totals(fields)
    res = hd.advance(fields, hd.GasModel(mu=0.0), hd.TimeParams(cfl=0.4, max_steps=100), mode=mode)
    mass1, mom1, energy1 = hd.conserved_totals(res.fields)
    mom_scale = params.rho0 * params.u0 * (2 * math.pi) ** 3
    assert abs(mass1 - mass0) / abs(mass0) < 1e-11
    assert abs(energy1 - energy0) / abs(energy0) < 1e-11
    assert max(abs(a - b) / max(abs(b), mom_scale) for a, b in zip(mom1, mom0)) < 1e-11


def test_decaying_turbulence_cascades_energy_to_small_scales(hd):
    """pkg/tests/test_acceptance.py:352-373: three eddy turnovers (t = 10) of
    viscous decay at 64^3 -- the high-wavenumber band fills, total KE falls."""
    params = hd.HitParams()
    spec = hd.GridSpec((64, 64, 64))
    fields = hd.make_initial_condition(spec, params, GAMMA_HIT, backend="numpy")
    before = hd.compute_spectrum(*_vel(fields))
    gas = hd.GasModel(mu=hd.viscosity_from_re_lambda(params))
    res = hd.advance(fields, gas, hd.TimeParams(cfl=0.4, t_final=10.0))
    after = hd.compute_spectrum(*_vel(res.fields))
    assert res.t == 10.0
    assert float(np.sum(after.energy[16:])) > float(np.sum(before.energy[16:]))
    assert after.total() < before.total()


def test_fast_mode_ke_curve_tracks_exact(hd):
    """The north-star tolerance over a long march: 64^3 HIT, RK4, 100 steps; the
    fast arithmetic's kinetic-energy curve stays within 1e-11 of the bitwise-
    reference curve at every step and the final state within 1e-10 relative L2."""
    spec = hd.GridSpec((64, 64, 64))
    ic = hd.make_initial_condition(spec, hd.HitParams(), backend="numpy")
    gas = hd.GasModel(mu=0.006)
    tp = hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=100)
    ex = hd.advance(ic, gas, tp, mode="exact")
    fa = hd.advance(ic, gas, tp, mode="fast")
    ke_ex = np.array([r.kinetic_energy for r in ex.records])
    ke_fa = np.array([r.kinetic_energy for r in fa.records])
    assert np.max(np.abs(ke_fa - ke_ex) / ke_ex) < 1e-11
    a = ex.fields.interior().reshape(5, -1)
    b = fa.fields.interior().reshape(5, -1)
    rel = ((b - a).norm(dim=1) / a.norm(dim=1)).cpu().numpy()
    assert np.all(rel <= 1e-10), rel


@pytest.mark.parametrize("n", [(32, 32, 32), (64, 48, 24)])
def test_flux_kernel_variants_agree(hd, n):
    """The TMA-fed flux kernel (HD_OPT_FLUX_TMA), the register-prefetch z-marching
    kernel and the pointwise kernel compute the same viscous fluxes (fast mode: the
    compiler may contract their FMAs differently), so 2 fast-mode RK4 steps
    (enstrophy folded into the first flux kernel) agree to round-off."""
    spec = hd.GridSpec(n)
    rng = np.random.default_rng(9)
    shape = spec.interior_shape
    rho = torch.from_numpy(0.8 + 0.4 * rng.random(shape)).cuda()
    vel = [torch.from_numpy(0.3 * rng.standard_normal(shape)).cuda() for _ in range(3)]
    p = torch.from_numpy(0.8 + 0.4 * rng.random(shape)).cuda()
    fs = _from_prims(hd, spec, rho, *vel, p)
    gas = hd.GasModel(mu=0.02)
    outs = []
    for tma, zmarch in ((1, 1), (0, 1), (0, 0)):
        hd.release_plans()
        plan = hd.get_plan(spec, gas, mode="fast")
        plan.set_option(hd._lib.HD_OPT_FLUX_TMA, tma)
        plan.set_option(hd._lib.HD_OPT_FLUX_ZMARCH, zmarch)
        res = hd.advance(fs, gas, hd.TimeParams(scheme="rk4", cfl=0.3, max_steps=2), mode="fast")
        outs.append((res.fields.interior().cpu().numpy(), [r.enstrophy for r in res.records]))
    hd.release_plans()
    for other in (outs[1][0], outs[2][0]):
        rel = np.sqrt(((other - outs[0][0]) ** 2).reshape(5, -1).sum(1) /
                      (outs[0][0] ** 2).reshape(5, -1).sum(1))
        assert np.all(rel <= 1e-14), rel
    for other in outs[1:]:
        assert np.allclose(outs[0][1], other[1], rtol=1e-13)
