"""BASELINE.json's full size (512^3 HIT, mu 0.006, RK4, CFL 0.4) on the GPU, checked
through size-independent properties (the oracle would need hours here):

* fast vs exact (bitwise-reference) arithmetic after 2 steps: <= 1e-10 relative L2
  per conserved variable (the north-star tolerance), dt to 1e-12;
* mass and momentum conserved to round-off (periodic box, flux form);
* kinetic energy decays monotonically (viscous decay, no forcing).
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hd():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    free, _ = torch.cuda.mem_get_info()
    if free < 120e9:
        pytest.skip("needs ~120 GB of free device memory")
    import paper_2211_16718_b200 as hd

    hd._lib.load(require_cuda=True)
    return hd


def test_512_fast_vs_exact_and_invariants(hd):
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
    hd.release_plans()
