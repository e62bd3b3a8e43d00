"""Largest single-GPU block of the 1024^3 / 4-GPU configuration: 1024 x 1024 x 256
(278 M ghosted points per field; workspace offsets beyond 2^31 elements), smooth
periodic state, a few fast-mode RK4 steps: finite, mass conserved, step rate.

    python tools/large_probe.py [--nz 256] [--steps 2]
"""
import argparse
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2211_16718_b200 as hd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nz", type=int, default=256)
ap.add_argument("--steps", type=int, default=2)
a = ap.parse_args()
spec = hd.GridSpec((1024, 1024, a.nz), (2 * math.pi, 2 * math.pi, 2 * math.pi * a.nz / 1024))
fs = hd.FieldSet.zeros(spec)
it = fs.interior()
z = torch.arange(a.nz, dtype=torch.float64, device="cuda")[:, None, None] * (2 * math.pi / a.nz)
y = torch.arange(1024, dtype=torch.float64, device="cuda")[None, :, None] * (2 * math.pi / 1024)
x = torch.arange(1024, dtype=torch.float64, device="cuda")[None, None, :] * (2 * math.pi / 1024)
it[0] = 1.0 + 0.1 * torch.sin(x) * torch.cos(y)
it[1] = it[0] * 0.3 * torch.sin(y + z)
it[2] = it[0] * 0.2 * torch.cos(x)
it[3] = it[0] * 0.1 * torch.sin(x + y)
it[4] = 2.5 + 0.5 * (it[1] ** 2 + it[2] ** 2 + it[3] ** 2) / it[0]
del x, y, z
m0 = float(it[0].sum()) * spec.cell_volume()
gas = hd.GasModel(mu=0.006)
hd.advance(fs, gas, hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=1))  # warm-up (plan, kernels)
torch.cuda.synchronize()
t0 = time.perf_counter()
res = hd.advance(fs, gas, hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=a.steps))
torch.cuda.synchronize()
el = time.perf_counter() - t0
body = res.fields.interior()
out = {"grid": list(spec.n), "ghosted_points": spec.total_points,
       "workspace_elements": 38 * spec.total_points, "finite": bool(torch.isfinite(body).all()),
       "mass_rel_change": abs(res.records[-1].mass - m0) / m0,
       "ms_per_step": 1e3 * el / a.steps, "pt_step_per_s": spec.interior_points * a.steps / el,
       "peak_mem_gb": torch.cuda.max_memory_allocated() / 1e9}
print(json.dumps(out))
assert out["finite"] and out["mass_rel_change"] < 1e-12
