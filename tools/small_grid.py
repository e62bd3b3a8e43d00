"""Step time of small grids, eager march vs CUDA-graph march (launch-bound regime).

    python tools/small_grid.py [--sizes 32,64,128] [--steps 41]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2211_16718_b200 as hd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", default="32,64,128")
ap.add_argument("--steps", type=int, default=41)
a = ap.parse_args()
out = {}
for n in (int(s) for s in a.sizes.split(",")):
    spec = hd.GridSpec((n,) * 3)
    ic = hd.make_initial_condition(spec, hd.HitParams(), backend="numpy")
    gas = hd.GasModel(mu=0.006)
    row = {}
    for mode_name, env in (("eager", "1"), ("graph", "0")):
        os.environ["HD_NO_GRAPH"] = env
        tp = hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=a.steps)
        hd.advance(ic, gas, tp)  # warm-up (plan, kernels)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = hd.advance(ic, gas, tp)
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        row[mode_name + "_ms_per_step"] = 1e3 * el / a.steps
        row[mode_name + "_pt_step_per_s"] = n ** 3 * a.steps / el
    out[n] = row
print(json.dumps(out, indent=1))
