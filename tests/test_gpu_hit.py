"""The GPU (torch/cuFFT) HIT initial condition -- the IC of every bench line and
of the 512^3/1024^3 configurations -- against the properties the reference
pins for its own synthesis (pkg/tests/test_hit.py:48-75, hit.py:93-139):

* every populated shell 1..n/2-1 carries exactly the target spectrum E(k)
  (1e-12), the mean shell holds nothing and shells >= n/2 only round-off;
* the field is solenoidal: max |k . c(k)| < 1e-12 u0 k0;
* KE is the isotropic value 3/2 u0^2 = 0.135 up to shell truncation;
* rho = rho0 and p = rho0/gamma everywhere (hit.py:210-236);
* deterministic for a seed, different for another seed.
"""

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


@pytest.mark.parametrize("n", [32, 64, 256, 512])
def test_torch_ic_shells_match_target(hd, n):
    P = hd.HitParams()
    u, v, w = hd.synthesize_velocity(n, P, "torch")
    table = hd.compute_spectrum(u, v, w)
    want = hd.target_spectrum(np.arange(1, n // 2, dtype=np.float64))
    got = table.energy[1:n // 2]
    # shells whose target lies well above the transform's absolute round-off
    # (~3e-26 at n <= 512; at n = 32 that is every shell, as in the reference
    # test) match to 1e-12; the far tail only to that round-off
    above = want > 1e-13
    np.testing.assert_allclose(got[above], want[above], rtol=1e-12, atol=0.0)
    assert np.all(np.abs(got[~above] - want[~above]) < 1e-24)
    assert table.energy[0] < 1e-30
    assert np.all(table.energy[n // 2:] < 1e-20)


@pytest.mark.parametrize("n", [32, 512])
def test_torch_ic_is_solenoidal(hd, n):
    P = hd.HitParams()
    u, v, w = hd.synthesize_velocity(n, P, "torch")
    assert u.dtype == torch.float64 and u.is_cuda
    assert hd.spectral_divergence(u, v, w) < 1e-12 * P.u0 * P.k0


@pytest.mark.parametrize("n", [64, 512])
def test_torch_ic_kinetic_energy(hd, n):
    P = hd.HitParams()
    u, v, w = hd.synthesize_velocity(n, P, "torch")
    ke = 0.5 * float((u * u + v * v + w * w).mean())
    assert ke == pytest.approx(1.5 * P.u0 ** 2, rel=0.02)
    # Parseval: the shell sum is the same KE
    assert hd.compute_spectrum(u, v, w).total() == pytest.approx(ke, rel=1e-10)


def test_torch_ic_state(hd):
    n = 64
    P = hd.HitParams()
    fs = hd.make_initial_condition(hd.GridSpec((n, n, n)), P, backend="torch")
    it = fs.interior()
    assert bool((it[0] == P.rho0).all())
    v2 = (it[1] ** 2 + it[2] ** 2 + it[3] ** 2) / it[0] ** 2
    p = 0.4 * (it[4] - 0.5 * it[0] * v2)
    assert torch.allclose(p, torch.full_like(p, P.rho0 / 1.4), rtol=1e-12, atol=0)
    # ghosts start zero; the first rhs fills them (hit.py:210-236)
    assert float(fs.data.abs().sum()) == pytest.approx(float(it.abs().sum()), rel=1e-12)


def test_torch_ic_seed(hd):
    a = hd.synthesize_velocity(32, hd.HitParams(), "torch")[0]
    b = hd.synthesize_velocity(32, hd.HitParams(), "torch")[0]
    c = hd.synthesize_velocity(32, hd.HitParams(seed=99), "torch")[0]
    assert torch.equal(a, b) and not torch.equal(a, c)


def test_spectral_divergence_backends_agree(hd):
    u, v, w = hd.synthesize_velocity(16, hd.HitParams(), "numpy")
    a = hd.spectral_divergence(u, v, w)
    t = [torch.from_numpy(x).cuda() for x in (u, v, w)]
    b = hd.spectral_divergence(*t)
    assert a < 1e-12 and b < 1e-12
