"""Does a memory-bound kernel (viscous RHS) co-run with a compute-bound sweep on a second stream?

    HD_LIB=... python tools/overlap_probe.py --n 512
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
a = ap.parse_args()
spec = hd.GridSpec((a.n,) * 3)
ic = hd.make_initial_condition(spec, hd.HitParams(), backend="torch")
gas = hd.GasModel(mu=0.006)
plan = hd.get_plan(spec, gas)
hd.fill_ghosts_periodic(ic)
inc = plan.fields(hd._lib.HD_BUF_INC, 5)
inc2 = torch.zeros_like(ic.data)
A = torch.cuda.current_stream()
B = torch.cuda.Stream(priority=-1)
e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e[0].record()
    for _ in range(reps):
        fn()
    e[1].record()
    torch.cuda.synchronize()
    return e[0].elapsed_time(e[1]) / reps


out = {}
for dim in (0, 1, 2):
    out[f"sweep{dim}"] = timed(lambda: plan.hyper_sweep(dim, ic.data, inc, dim != 0))
out["visc"] = timed(lambda: plan.parabolic_rhs(ic.data, inc2))


def both(dim):
    def fn():
        ev = torch.cuda.Event()
        ev.record(A)
        B.wait_event(ev)
        with torch.cuda.stream(B):
            plan.parabolic_rhs(ic.data, inc2)
        plan.hyper_sweep(dim, ic.data, inc, dim != 0)
        ev2 = torch.cuda.Event()
        ev2.record(B)
        A.wait_event(ev2)
    return fn


def both_sweep_first(dim):
    def fn():
        ev = torch.cuda.Event()
        ev.record(A)
        B.wait_event(ev)
        plan.hyper_sweep(dim, ic.data, inc, dim != 0)
        with torch.cuda.stream(B):
            plan.parabolic_rhs(ic.data, inc2)
        ev2 = torch.cuda.Event()
        ev2.record(B)
        A.wait_event(ev2)
    return fn


for dim in (0, 1, 2):
    out[f"sweep{dim}+visc concurrent"] = timed(both(dim))
    out[f"sweep{dim} first +visc concurrent"] = timed(both_sweep_first(dim))
print(json.dumps(out))
