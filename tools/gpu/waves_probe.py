"""Step time vs the sweep segment heuristic (HD_OPT_SWEEP_WAVES) on per-GPU block
shapes of the decomposed runs (periodic stand-ins), e.g. 256x256x64 = 256^3 on 4 GPUs."""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2211_16718_b200 as hd  # noqa: E402

shapes = [tuple(int(v) for v in s.split("x")) for s in sys.argv[1].split(",")]
waves_list = [int(w) for w in sys.argv[2].split(",")]
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
    row = {"shape": shape}
    for w in waves_list:
        hd.release_plans()
        hd.get_plan(spec, gas).set_option(hd._lib.HD_OPT_SWEEP_WAVES, w)
        r = hd.advance(fs, gas, hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=2))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        r = hd.advance(r.fields, gas, hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=6))
        e1.record()
        torch.cuda.synchronize()
        row[f"w{w}_ms"] = round(e0.elapsed_time(e1) / 6, 3)
    print(json.dumps(row), flush=True)
