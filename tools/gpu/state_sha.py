"""SHA-256 of the state after a few fast-mode RK4 steps (to check that a kernel
change is bitwise neutral): python tools/gpu/state_sha.py [n] [steps]"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2211_16718_b200 as hd  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
spec = hd.GridSpec((n,) * 3)
ic = hd.make_initial_condition(spec, hd.HitParams(), backend="torch")
r = hd.advance(ic, hd.GasModel(mu=0.006), hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=steps), mode="fast")
print(n, steps, hashlib.sha256(r.fields.interior().cpu().numpy().tobytes()).hexdigest(), r.t)
