"""How far fast mode sits from exact mode (the reference's arithmetic): relative L2
per conserved variable after N RK4 steps from the HIT IC, and the dt drift."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import paper_2211_16718_b200 as hd  # noqa: E402

out = {}
for n, steps in ((32, 20), (64, 20), (128, 4)):
    spec = hd.GridSpec((n,) * 3)
    ic = hd.make_initial_condition(spec, hd.HitParams(), backend="torch")
    tp = hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=steps)
    ra = hd.advance(ic, hd.GasModel(mu=0.006), tp, mode="exact")
    rb = hd.advance(ic, hd.GasModel(mu=0.006), tp, mode="fast")
    a = ra.fields.interior().cpu().numpy().reshape(5, -1)
    b = rb.fields.interior().cpu().numpy().reshape(5, -1)
    rel = np.sqrt(((b - a) ** 2).sum(1) / (a ** 2).sum(1))
    dts = max(abs(x.dt - y.dt) / x.dt for x, y in zip(ra.records, rb.records))
    out[f"{n}^3x{steps}"] = {"rel_l2": [float(f"{v:.3e}") for v in rel], "max_dt_rel": float(f"{dts:.3e}")}
    hd.release_plans()
print(json.dumps(out))
