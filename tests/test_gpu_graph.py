"""The CUDA-graph march (timeint._DeviceMarch._run_graph): chunks of steps
replayed from one graph must give exactly the eager march -- state, every
step record, and the step/stage of a StepError raised mid-chunk."""

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


def _run(hd, monkeypatch, graph, fs, gas, tp, mode):
    monkeypatch.setenv("HD_NO_GRAPH", "0" if graph else "1")
    return hd.advance(fs, gas, tp, mode=mode)


@pytest.mark.parametrize("mode", ["exact", "fast"])
@pytest.mark.parametrize("stepping", [dict(cfl=0.4), dict(dt=0.01)])
def test_graph_march_equals_eager(hd, monkeypatch, mode, stepping):
    spec = hd.GridSpec((32, 32, 32))
    ic = hd.make_initial_condition(spec, hd.HitParams(), backend="numpy")
    gas = hd.GasModel(mu=0.006)
    tp = hd.TimeParams(scheme="rk4", max_steps=22, **stepping)  # step 0 + 2 chunks of 8 + 5 eager
    a = _run(hd, monkeypatch, False, ic, gas, tp, mode)
    b = _run(hd, monkeypatch, True, ic, gas, tp, mode)
    assert torch.equal(a.fields.data, b.fields.data)
    assert a.t == b.t and len(a.records) == len(b.records) == 22
    for ra, rb in zip(a.records, b.records):
        assert (ra.step, ra.t, ra.dt, ra.mass, ra.energy, ra.kinetic_energy) == \
               (rb.step, rb.t, rb.dt, rb.mass, rb.energy, rb.kinetic_energy)
        # graph chunks run the stand-alone enstrophy pass, the eager march folds it
        # into the next step's flux kernel (fast mode: different reciprocals)
        assert np.isclose(ra.enstrophy, rb.enstrophy, rtol=1e-13, atol=0)


def test_graph_march_step_error_mid_chunk(hd, monkeypatch):
    """A fixed dt slightly too large: the state blows up after several steps;
    the graph path must name the same step and stage as the eager path."""
    n = 16
    spec = hd.GridSpec((n, n, n))
    fs = hd.FieldSet.zeros(spec)
    x = torch.arange(n, dtype=torch.float64, device="cuda") * (2 * np.pi / n)
    w = 0.5 * torch.sin(x)[:, None, None]
    fs.interior()[0] = 1.0
    fs.interior()[3] = w
    fs.interior()[4] = 2.5 + 0.5 * w * w
    gas = hd.GasModel()
    found = None
    for dt in (1.2, 1.0, 0.9, 0.8, 0.7, 0.6, 0.5):
        tp = hd.TimeParams(scheme="rk4", dt=dt, max_steps=40)
        try:
            _run(hd, monkeypatch, False, fs, gas, tp, "exact")
        except hd.StepError as e:
            if e.step >= 3:
                found = (tp, e.step, e.stage)
                break
    assert found is not None, "no fixed dt produced a late blow-up"
    tp, step, stage = found
    with pytest.raises(hd.StepError) as ei:
        _run(hd, monkeypatch, True, fs, gas, tp, "exact")
    assert (ei.value.step, ei.value.stage) == (step, stage)
