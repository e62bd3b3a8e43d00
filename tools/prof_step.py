"""Profiling driver: W warm-up + K RK4 steps of the n^3 HIT problem (for ncu).

    python tools/prof_step.py --n 512 --steps 1 --warmup 1 [--mode fast]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2211_16718_b200 as hd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--warmup", type=int, default=1)
ap.add_argument("--mode", default="fast")
a = ap.parse_args()
hd.set_mode(a.mode)
spec = hd.GridSpec((a.n,) * 3)
ic = hd.make_initial_condition(spec, hd.HitParams(), backend="torch" if a.n > 128 else "numpy")
gas = hd.GasModel(mu=0.006)
res = hd.advance(ic, gas, hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=a.warmup))
torch.cuda.synchronize()
res = hd.advance(res.fields, gas, hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=a.steps))
torch.cuda.synchronize()
print("steps", res.steps, "t", res.t, "ke", res.records[-1].kinetic_energy)
