"""Flux-kernel variants at n^3 (HD_OPT_FLUX_TMA 0/1/2): time per launch (CUDA events) and a
full-step time."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2211_16718_b200 as hd  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
spec = hd.GridSpec((n,) * 3)
ic = hd.make_initial_condition(spec, hd.HitParams(), backend="torch")
gas = hd.GasModel(mu=0.006)
hd.fill_ghosts_periodic(ic)
out = {"n": n}
for opt in (1, 0):
    hd.release_plans()
    plan = hd.get_plan(spec, gas)
    plan.set_option(hd._lib.HD_OPT_FLUX_TMA, opt)
    plan.timer_enable(True)
    r = hd.advance(ic, gas, hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=2))
    plan.timer_read()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    r = hd.advance(r.fields, gas, hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=5))
    e1.record()
    torch.cuda.synchronize()
    kt = plan.timer_read()
    out[f"opt{opt}"] = {"step_ms": e0.elapsed_time(e1) / 5,
                        "flux_ms": kt["gradflux"][0] / max(kt["gradflux"][1], 1),
                        "ens": r.records[-1].enstrophy}
    del r
print(json.dumps(out))
