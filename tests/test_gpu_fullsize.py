"""The benchmark configurations (BASELINE.json configs 2-4: 128^3, 256^3, 512^3 HIT,
mu 0.006, RK4, CFL 0.4) on the GPU against the C oracle run on every host thread:

* exact mode: final state and every dt bitwise equal to the oracle (which is
  itself bitwise equal to the reference, tests/test_oracle_golden.py);
* fast mode: <= 1e-10 relative L2 per conserved variable (the north-star
  tolerance), dt to 1e-12;
* KE and enstrophy of each step against the oracle's state (1e-11).

128^3 runs 2 steps and 256^3 1 step from the reference's own IC synthesis
(numpy backend, bit-identical to hit.py); 512^3 runs 1 step from the GPU
synthesis the bench uses (its interior is handed to the oracle), gated on host
RAM (~75 GB for the oracle) and device memory.  A 2-step 512^3 fast-vs-exact
run adds the invariants of the periodic flux-form scheme.
"""

import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hd():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2211_16718_b200 as hd

    hd._lib.load(require_cuda=True)
    return hd


def _host_ram_gb() -> float:
    return os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 1e9


def _need_device_gb(gb: float) -> None:
    free, _ = torch.cuda.mem_get_info()
    if free < gb * 1e9:
        pytest.skip(f"needs ~{gb:.0f} GB of free device memory")


def _oracle_run(oracle, ic_interior: np.ndarray, n: int, steps: int):
    """(final interior, dts, KE per step, enstrophy per step) of the C oracle."""
    oracle.set_num_threads(len(os.sched_getaffinity(0)))
    P = oracle.Problem(n=(n, n, n), mu=0.006)
    U = oracle.from_interior(ic_interior, P)
    dts, ke, ens = [], [], []
    for _ in range(steps):
        dts += list(oracle.advance(U, P, 1, cfl=0.4))
        body = oracle.interior(U, P)
        ke.append(float(np.mean(0.5 * ((body[1] / body[0]) ** 2 + (body[2] / body[0]) ** 2 +
                                        (body[3] / body[0]) ** 2))))
        ens.append(oracle.enstrophy(U, P))
    return np.ascontiguousarray(oracle.interior(U, P)), dts, ke, ens


def _check(hd, ic, want, dts, ke, ens, steps):
    gas = hd.GasModel(mu=0.006)
    tp = hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=steps)
    for mode in ("exact", "fast"):
        hd.release_plans()
        res = hd.advance(ic, gas, tp, mode=mode)
        got = res.fields.interior().cpu().numpy()
        got_dt = [r.dt for r in res.records]
        if mode == "exact":
            assert np.array_equal(got, want), "exact mode differs from the oracle"
            assert got_dt == dts
        else:
            rel = np.sqrt(((got - want) ** 2).reshape(5, -1).sum(1)) / \
                np.sqrt((want ** 2).reshape(5, -1).sum(1))
            assert np.all(rel <= 1e-10), rel
            assert np.allclose(got_dt, dts, rtol=1e-12, atol=0)
        assert np.allclose([r.kinetic_energy for r in res.records], ke, rtol=1e-11, atol=0)
        assert np.allclose([r.enstrophy for r in res.records], ens, rtol=1e-11, atol=0)
        del res, got
    hd.release_plans()


@pytest.mark.parametrize("n,steps", [(128, 2), (256, 1)])
def test_hit_config_matches_oracle(hd, oracle, n, steps):
    _need_device_gb((n + 6) ** 3 * 400 / 1e9)  # two plans' workspaces + the IC
    spec = hd.GridSpec((n, n, n))
    ic = hd.make_initial_condition(spec, hd.HitParams(), backend="numpy")  # hit.py's own stream
    want, dts, ke, ens = _oracle_run(oracle, ic.interior().cpu().numpy(), n, steps)
    _check(hd, ic, want, dts, ke, ens, steps)


def test_512_matches_oracle(hd, oracle):
    if _host_ram_gb() < 100:
        pytest.skip("the 512^3 oracle step needs ~75 GB of host RAM")
    _need_device_gb(110)
    n = 512
    spec = hd.GridSpec((n, n, n))
    ic = hd.make_initial_condition(spec, hd.HitParams(), backend="torch")  # the bench's IC
    want, dts, ke, ens = _oracle_run(oracle, ic.interior().cpu().numpy(), n, 1)
    _check(hd, ic, want, dts, ke, ens, 1)


def test_512_fast_vs_exact_and_invariants(hd):
    _need_device_gb(120)
    n = 512
    spec = hd.GridSpec((n, n, n))
    ic = hd.make_initial_condition(spec, hd.HitParams(), backend="torch")
    gas = hd.GasModel(mu=0.006)
    tp = hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=2)
    hd.release_plans()
    ex = hd.advance(ic, gas, tp, mode="exact")
    exact = ex.fields.interior().clone()
    ex_recs = ex.records
    del ex
    hd.release_plans()
    torch.cuda.empty_cache()
    fa = hd.advance(ic, gas, tp, mode="fast")
    fast = fa.fields.interior()
    diff = (fast - exact).reshape(5, -1)
    ref = exact.reshape(5, -1)
    rel = (diff.norm(dim=1) / ref.norm(dim=1)).cpu().numpy()
    assert np.all(rel <= 1e-10), rel
    for a, b in zip(ex_recs, fa.records):
        assert abs(a.dt - b.dt) <= 1e-12 * a.dt
    # invariants of the periodic flux-form scheme (records: totals after each step)
    m0 = float(ic.interior()[0].sum()) * spec.cell_volume()
    for recs in (ex_recs, fa.records):
        for r in recs:
            assert abs(r.mass - m0) <= 1e-12 * m0
            assert max(abs(c) for c in r.momentum) <= 1e-11 * m0
        ke = [r.kinetic_energy for r in recs]
        assert ke[1] < ke[0]
        ens = [r.enstrophy for r in recs]
        assert np.all(np.isfinite(ens)) and ens[0] > 0.0
    hd.release_plans()
