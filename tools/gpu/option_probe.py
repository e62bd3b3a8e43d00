"""Step time and per-kernel times at n^3 for each value of one plan option
(hd_plan_set_option), e.g.  python tools/gpu/option_probe.py 512 X_STAGED 1,2"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2211_16718_b200 as hd  # noqa: E402

n = int(sys.argv[1])
opt = getattr(hd._lib, "HD_OPT_" + sys.argv[2])
values = [int(v) for v in sys.argv[3].split(",")]
spec = hd.GridSpec((n,) * 3)
ic = hd.make_initial_condition(spec, hd.HitParams(), backend="torch")
gas = hd.GasModel(mu=0.006)
out = {"n": n, "option": sys.argv[2]}
plan = None
for rep in range(2):
    for val in values:
        plan = None
        hd.release_plans()
        plan = hd.get_plan(spec, gas)
        plan.set_option(opt, val)
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
        row = {"step_ms": round(e0.elapsed_time(e1) / 5, 3),
               **{k: round(v[0] / v[1], 3) for k, v in kt.items() if v[1]}, "ke": r.records[-1].kinetic_energy}
        out[f"{val}_rep{rep}"] = row
        del r
print(json.dumps(out))
