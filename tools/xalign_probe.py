"""x-sweep time per point: 512^3 (ghosted rows of 518 doubles: alternate 16-byte
alignment) vs 510 x 512 x 512 (rows of 516: every row 32-byte aligned)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2211_16718_b200 as hd  # noqa: E402

out = {}
for n0 in (512, 510):
    spec = hd.GridSpec((n0, 512, 512))
    fs = hd.FieldSet.zeros(spec)
    it = fs.interior()
    it[0] = 1.0
    it[1] = 0.1 * torch.rand_like(it[1])
    it[4] = 2.5
    hd.fill_ghosts_periodic(fs)
    plan = hd.get_plan(spec, hd.GasModel())
    inc = plan.fields(hd._lib.HD_BUF_INC, 5)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    plan.hyper_sweep(0, fs.data, inc, False)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        plan.hyper_sweep(0, fs.data, inc, False)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    out[n0] = {"ms": ms, "ns_per_pt": ms * 1e6 / spec.interior_points}
    hd.release_plans()
    del fs
    torch.cuda.empty_cache()
print(json.dumps(out))
