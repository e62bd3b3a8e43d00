"""Time the individual kernels of one RK stage at n^3 (CUDA events), for variant comparisons.

    HD_LIB=path/to/libhd.so python tools/sweep_bench.py --n 512
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
ap.add_argument("--mode", default="fast")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--mu", type=float, default=0.006)
a = ap.parse_args()
hd.set_mode(a.mode)
spec = hd.GridSpec((a.n,) * 3)
ic = hd.make_initial_condition(spec, hd.HitParams(), backend="torch" if a.n > 128 else "numpy")
gas = hd.GasModel(mu=a.mu)
plan = hd.get_plan(spec, gas)
hd.fill_ghosts_periodic(ic)
inc = plan.fields(hd._lib.HD_BUF_INC, 5)
out = {"lib": os.environ.get("HD_LIB", "default"), "n": a.n, "mode": a.mode}
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for dim in range(3):
    plan.hyper_sweep(dim, ic.data, inc, True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(a.reps):
        plan.hyper_sweep(dim, ic.data, inc, True)
    e1.record()
    torch.cuda.synchronize()
    out[f"sweep{dim}_ms"] = e0.elapsed_time(e1) / a.reps
plan.parabolic_rhs(ic.data, inc)
torch.cuda.synchronize()
e0.record()
for _ in range(a.reps):
    plan.parabolic_rhs(ic.data, inc)
e1.record()
torch.cuda.synchronize()
out["viscous_ms"] = e0.elapsed_time(e1) / a.reps
print(json.dumps(out))
tp = hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=1)
res = hd.advance(ic, gas, tp)
torch.cuda.synchronize()
tp = hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=3)
e0.record()
res = hd.advance(res.fields, gas, tp)
e1.record()
torch.cuda.synchronize()
out["step_ms"] = e0.elapsed_time(e1) / 3
out["pt_step_per_s"] = a.n ** 3 / (out["step_ms"] / 1e3)
print(json.dumps(out))
