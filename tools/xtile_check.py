"""x sweep: thread-per-cell tile kernel (HD_XTILE=1) against the staged marching
kernel -- bitwise on a fast-mode march (incl. ragged error paths), and timing.

    python tools/xtile_check.py [--n 512] [--steps 3]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2211_16718_b200 as hd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--steps", type=int, default=3)
a = ap.parse_args()
spec = hd.GridSpec((a.n,) * 3)
ic = hd.make_initial_condition(spec, hd.HitParams(), backend="torch" if a.n > 128 else "numpy",
                               device="cuda")
gas = hd.GasModel(mu=0.006)
out = {}
res = {}
for tag, env in (("staged", None), ("tile", "1")):
    if env:
        os.environ["HD_XTILE"] = env
    else:
        os.environ.pop("HD_XTILE", None)
    tp = hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=a.steps)
    hd.advance(ic, gas, hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=1), mode="fast")
    torch.cuda.synchronize()
    plan = hd.get_plan(spec, gas, mode="fast")
    plan.timer_read()
    plan.timer_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = hd.advance(ic, gas, tp, mode="fast")
    e1.record()
    torch.cuda.synchronize()
    kt = plan.timer_read()
    plan.timer_enable(False)
    res[tag] = r.fields.data.clone()
    out[tag] = {"ms_per_step": e0.elapsed_time(e1) / a.steps,
                "kernels_ms": {k: round(v[0] / max(v[1], 1), 3) for k, v in kt.items() if v[1]}}
out["bitwise"] = bool(torch.equal(res["staged"], res["tile"]))
out["max_abs_diff"] = float((res["staged"] - res["tile"]).abs().max())
print(json.dumps(out))
