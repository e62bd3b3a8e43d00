"""Do sector-aligned rows pay for the y/z sweeps?  Plain y and z sweeps
(hd_hyper_sweep) on a 506x512x512 box (row pitch 512 doubles, a multiple of 4),
with the state and increment buffers starting on a 256-byte boundary (interior
rows then start 24 bytes into a sector) or 8 bytes past it (interior rows
sector-aligned).  Prints ms per sweep for each placement."""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2211_16718_b200 as hd  # noqa: E402

shape = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "506x512x512").split("x"))
spec = hd.GridSpec(shape, tuple(2 * math.pi * s / shape[0] for s in shape))
gas = hd.GasModel(mu=0.006)
plan = hd.get_plan(spec, gas)
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
hd.fill_ghosts_periodic(fs) if hasattr(hd, "fill_ghosts_periodic") else None
src = fs.data.reshape(-1)
n = src.numel()
res = {"shape": shape}
for off in (0, 1, 0, 1):
    ubuf = torch.empty(n + 32, dtype=torch.float64, device="cuda")
    ibuf = torch.zeros(n + 32, dtype=torch.float64, device="cuda")
    u = ubuf[off:off + n]
    inc = ibuf[off:off + n]
    u.copy_(src)
    row = {}
    for dim in (1, 2):
        plan.hyper_sweep(dim, u, inc, True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(5):
            plan.hyper_sweep(dim, u, inc, True)
        e1.record()
        torch.cuda.synchronize()
        row[f"dim{dim}_ms"] = round(e0.elapsed_time(e1) / 5, 4)
    row["u_mod32"] = u.data_ptr() % 32
    res.setdefault(f"off{off}", []).append(row)
    del ubuf, ibuf, u, inc
print(json.dumps(res))
