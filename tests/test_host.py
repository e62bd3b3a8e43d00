"""Host-side logic that runs without a GPU: parameter records, stepper
composition with scalar fake right-hand sides (the reference's own anchors,
pkg/tests/test_timeint.py:74-103, test_acceptance.py:42-66), error-key
decoding, solution files, the initial condition."""

import hashlib
import math

import numpy as np
import pytest
import torch

import paper_2211_16718_b200 as hd
from paper_2211_16718_b200.plan import decode_key, error_from_key


def _scalar(value):
    fs = hd.FieldSet.zeros(hd.GridSpec((1, 1, 1)), device="cpu")
    fs.interior()[:] = value
    return fs


def _val(fs):
    return float(fs.interior()[0, 0, 0, 0])


def _decay(f):
    return hd.FieldSet(f.spec, f.layout, -f.data)


def test_rk_amplification_factors():
    assert abs(_val(hd.rk3_tvd_step(_scalar(1.0), 0.1, _decay)) - 0.9048333333333334) < 1e-14
    assert abs(_val(hd.rk4_step(_scalar(1.0), 0.1, _decay)) - 0.9048375) < 1e-14


@pytest.mark.parametrize("name,min_order", [("rk3", 2.7), ("rk4", 3.7)])
def test_temporal_order(name, min_order):
    stepper = hd.STEPPERS[name]
    rhs = lambda f: hd.FieldSet(f.spec, f.layout, -(f.data * f.data))  # y' = -y^2, y = 1/(1+t)
    errs = []
    for steps in (20, 40):
        fs = _scalar(1.0)
        for _ in range(steps):
            fs = stepper(fs, 1.0 / steps, rhs)
        errs.append(abs(_val(fs) - 0.5))
    assert math.log2(errs[0] / errs[1]) > min_order


@pytest.mark.parametrize("kwargs", [
    dict(scheme="rk5", dt=0.1, max_steps=1), dict(dt=0.1, cfl=0.4, max_steps=1),
    dict(max_steps=1), dict(dt=0.1), dict(dt=-1.0, max_steps=1), dict(cfl=0.0, max_steps=1),
    dict(dt=0.1, t_final=-1.0), dict(dt=0.1, max_steps=-2), dict(cfl=0.4, cfl_mode="min", max_steps=1),
])
def test_time_params_validation(kwargs):
    with pytest.raises(ValueError):
        hd.TimeParams(**kwargs)


def test_parameter_records_validate():
    with pytest.raises(ValueError):
        hd.GasModel(gamma=1.0)
    with pytest.raises(ValueError):
        hd.WenoParams(power=0)
    with pytest.raises(ValueError):
        hd.GridSpec((8, 8, 8), ghost_width=2)
    assert hd.GasModel(mu=0.01, visc_scale=2.0).effective_mu == 0.02
    spec = hd.GridSpec((4, 5, 6))
    assert spec.shape == (12, 11, 10) and spec.total_points == 1320
    assert hd.linear_index(spec, -3, -3, -3) == 0


def test_error_key_decoding():
    spec = hd.GridSpec((8, 8, 8))
    point = hd.linear_index(spec, 2, 3, 4)
    # step 5 (0-based 4), RK stage 2 (slot 3), pressure (code 2)
    key = ((4 * 8 + 3) << 36) | (2 << 34) | point
    assert decode_key(key) == (4, 3, 2, point)
    err = error_from_key(key, spec)
    assert isinstance(err, hd.StepError) and err.step == 5 and err.stage == 2
    assert isinstance(err.__cause__.__cause__, hd.InvalidStateError)
    assert err.__cause__.__cause__.where == (4 + 3, 3 + 3, 2 + 3)
    # slot 0 / 7 (CFL reduction, diagnostics) -> InvalidStateError, not StepError
    err = error_from_key(((4 * 8 + 7) << 36) | (1 << 34) | point, spec)
    assert isinstance(err, hd.InvalidStateError) and not isinstance(err, hd.StepError)
    # ... whose `where` is an interior index (cons_to_prim on fields.interior())
    assert err.where == (4, 3, 2)
    err = error_from_key((7 << 36) | (3 << 34), spec)
    assert "dt" in str(err)


def test_solution_file_roundtrip(tmp_path):
    spec = hd.GridSpec((6, 5, 4), length=(1.0, 2.0, 3.0))
    fs = hd.FieldSet.zeros(spec, device="cpu")
    fs.interior().copy_(torch.arange(5 * 120, dtype=torch.float64).view(5, 4, 5, 6))
    path = tmp_path / "s.bin"
    hd.write_solution(path, fs, 0.25)
    back, t = hd.read_solution(path, device="cpu")
    assert t == 0.25 and back.spec == spec
    assert torch.equal(back.interior(), fs.interior())
    raw = path.read_bytes()
    path.write_bytes(b"XXXXXXXX" + raw[8:])
    with pytest.raises(hd.SolutionFormatError):
        hd.read_solution(path, device="cpu")
    path.write_bytes(raw[:-8])
    with pytest.raises(hd.SolutionFormatError):
        hd.read_solution(path, device="cpu")


def test_reference_solution_file_is_readable(tmp_path):
    """HITDNS01 files written by the reference load unchanged (grid.py:272-325)."""
    import os
    import sys

    ref = "/root/reference/pkg/src"
    if not os.path.isdir(ref):
        pytest.skip("reference not mounted")
    sys.path.insert(0, ref)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nb")
    try:
        import hitdns
    finally:
        sys.path.remove(ref)
    rspec = hitdns.GridSpec((4, 6, 8))
    rfs = hitdns.FieldSet.zeros(rspec)
    rfs.interior()[...] = np.random.default_rng(1).random((5, 8, 6, 4))
    hitdns.write_solution(tmp_path / "r.bin", rfs, 1.5)
    back, t = hd.read_solution(tmp_path / "r.bin", device="cpu")
    assert t == 1.5 and np.array_equal(back.interior().numpy(), rfs.interior())


def test_initial_condition_matches_reference_bits(traj32_golden):
    ic = hd.make_initial_condition(hd.GridSpec((32, 32, 32)), hd.HitParams(), backend="numpy",
                                   device="cpu")
    digest = hashlib.sha256(ic.interior().numpy().tobytes()).hexdigest()
    assert digest == traj32_golden["ic_sha256"]
    u, v, w = (ic.interior()[a] / ic.interior()[0] for a in (1, 2, 3))
    spec = hd.compute_spectrum(u.numpy(), v.numpy(), w.numpy())
    assert abs(spec.total() - traj32_golden["ke"][0]) < 1e-12
    assert abs(hd.viscosity_from_re_lambda(hd.HitParams()) - 0.006) < 1e-15


def test_pointwise_physics_helpers():
    """physics.py:58-255 utilities on tensors: round trip, fluxes, positivity errors."""
    import paper_2211_16718_b200 as hd

    rng = np.random.default_rng(11)
    prim = np.stack([0.5 + rng.random(20), rng.standard_normal(20), rng.standard_normal(20),
                     rng.standard_normal(20), 0.5 + rng.random(20)], axis=-1)
    cons = hd.prim_to_cons(torch.from_numpy(prim), 1.4)
    back = hd.cons_to_prim(cons, 1.4)
    assert torch.allclose(back, torch.from_numpy(prim).to(back.device), rtol=1e-13, atol=1e-14)
    a = hd.sound_speed(back, 1.4).cpu().numpy()
    assert np.allclose(a, np.sqrt(1.4 * prim[:, 4] / prim[:, 0]), rtol=1e-14)
    f = hd.convective_flux(cons, 1, 1.4).cpu().numpy()
    c = cons.cpu().numpy()
    assert np.allclose(f[:, 0], c[:, 2], rtol=1e-14)
    assert np.allclose(f[:, 2], c[:, 2] * prim[:, 2] + prim[:, 4], rtol=1e-13)
    assert np.allclose(hd.max_wavespeed(cons, 0, 1.4).cpu().numpy(), np.abs(prim[:, 1]) + a, rtol=1e-13)
    g = torch.from_numpy(rng.standard_normal((4, 3, 3)))
    tau = hd.viscous_stress(g, 0.1).cpu()
    assert torch.allclose(tau, tau.transpose(-2, -1))
    assert torch.allclose(tau.diagonal(dim1=-2, dim2=-1).sum(-1), torch.zeros(4, dtype=torch.float64), atol=1e-15)
    bad = prim.copy()
    bad[3, 0] = -1.0
    with pytest.raises(hd.InvalidStateError):
        hd.cons_to_prim(hd.prim_to_cons(torch.from_numpy(bad), 1.4), 1.4)
    spec = hd.GridSpec((4, 4, 4))
    fs = hd.FieldSet.zeros(spec, device="cpu")
    fs.data.view(5, -1)[0] = 1.0
    fs.data.view(5, -1)[4] = 2.5
    rho, u, v, w, p = hd.decode_primitives(fs, 1.4)
    assert float(p.min()) == pytest.approx(1.0) and float(u.abs().max()) == 0.0
