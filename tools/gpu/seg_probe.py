"""Per-kernel times (plan timer) against a forced sweep segment count
(HD_OPT_SEGMENTS, all three sweeps alike; 0 = the plan's own choice) on a periodic
box of any shape, e.g.  python tools/gpu/seg_probe.py 512x512x512,256x256x64 0,1,2,3,4"""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2211_16718_b200 as hd  # noqa: E402

shapes = [tuple(int(v) for v in s.split("x")) for s in sys.argv[1].split(",")]
segs = [int(w) for w in sys.argv[2].split(",")]
extra = [tuple(int(v) for v in kv.split("=")) for kv in sys.argv[3:]]  # option=value pairs
gas = hd.GasModel(mu=0.006)
for shape in shapes:
    spec = hd.GridSpec(shape, tuple(2 * math.pi * s / shape[0] for s in shape))
    fs = hd.FieldSet.zeros(spec)
    it = fs.interior()
    z, y, x = torch.meshgrid(*(torch.arange(n, dtype=torch.float64, device="cuda") * (2 * math.pi / shape[0])
                               for n in (shape[2], shape[1], shape[0])), indexing="ij")
    it[0] = 1.0 + 0.1 * torch.sin(x + y)
    it[1] = it[0] * 0.3 * torch.sin(x) * torch.cos(y) * torch.cos(z)
    it[2] = -it[0] * 0.3 * torch.cos(x) * torch.sin(y) * torch.cos(z)
    it[3] = it[0] * 0.05 * torch.sin(2 * z)
    it[4] = 2.5 + 0.5 * (it[1] ** 2 + it[2] ** 2 + it[3] ** 2) / it[0]
    del x, y, z
    for seg in segs:
        hd.release_plans()
        plan = hd.get_plan(spec, gas)
        plan.set_option(hd._lib.HD_OPT_SEGMENTS, seg)
        for k, v in extra:
            plan.set_option(k, v)
        r = hd.advance(fs, gas, hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=2))
        plan.timer_enable(True)
        plan.timer_read()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        r = hd.advance(r.fields, gas, hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=4))
        e1.record()
        torch.cuda.synchronize()
        kt = plan.timer_read()
        plan.timer_enable(False)
        row = {"shape": shape, "seg": seg, "step_ms": round(e0.elapsed_time(e1) / 4, 3),
               **{k: round(v[0] / v[1], 4) for k, v in kt.items() if v[1]}}
        print(json.dumps(row), flush=True)
        del r, plan
