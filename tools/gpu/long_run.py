"""A long fast-mode run at the benchmark size: 512^3 HIT IC, RK4 CFL 0.4, mu 0.006,
N steps through hd.advance; reports the diagnostics' evolution and conservation."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2211_16718_b200 as hd  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
spec = hd.GridSpec((n,) * 3)
ic = hd.make_initial_condition(spec, hd.HitParams(), backend="torch")
m0 = float(ic.interior()[0].sum()) * spec.cell_volume()
e0 = float(ic.interior()[4].sum()) * spec.cell_volume()
torch.cuda.synchronize()
t0 = time.perf_counter()
r = hd.advance(ic, hd.GasModel(mu=0.006), hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=steps))
torch.cuda.synchronize()
el = time.perf_counter() - t0
it = r.fields.interior()
m1 = float(it[0].sum()) * spec.cell_volume()
e1 = float(it[4].sum()) * spec.cell_volume()
rec = r.records
print(json.dumps({
    "grid": n, "steps": steps, "t": r.t, "wall_s": el, "finite": bool(torch.isfinite(it).all()),
    "mass_rel_change": abs(m1 - m0) / abs(m0), "energy_rel_change": abs(e1 - e0) / abs(e0),
    "ke": [rec[0].kinetic_energy, rec[len(rec) // 2].kinetic_energy, rec[-1].kinetic_energy],
    "enstrophy": [rec[0].enstrophy, rec[len(rec) // 2].enstrophy, rec[-1].enstrophy],
    "dt_first_last": [rec[0].dt, rec[-1].dt]}))
