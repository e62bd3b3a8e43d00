"""Clock and board power while one kernel kind runs back to back (~2 s each) at 512^3:
nvidia-smi sampled every 100 ms during the loop.  Shows which kernels hold the
1 kW cap (sw_power_cap) and at what SM clock."""
import json
import os
import statistics
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2211_16718_b200 as hd  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
spec = hd.GridSpec((n,) * 3)
ic = hd.make_initial_condition(spec, hd.HitParams(), backend="torch")
gas = hd.GasModel(mu=0.006)
hd.fill_ghosts_periodic(ic)
plan = hd.get_plan(spec, gas)
inc = plan.fields(hd._lib.HD_BUF_INC, 5)
L = hd._lib.load()
import ctypes  # noqa: E402

stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
kinds = {
    "sweep_x": lambda: plan.hyper_sweep(0, ic.data, inc, False),
    "sweep_y": lambda: plan.hyper_sweep(1, ic.data, inc, True),
    "sweep_z": lambda: plan.hyper_sweep(2, ic.data, inc, True),
    "flux_tma": lambda: L.hd_viscous_fluxes(plan.h, ctypes.c_void_p(ic.data.data_ptr()), stream),
}
out = {}
for name, fn in kinds.items():
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    reps = max(1, int(2500 / e0.elapsed_time(e1)))
    smi = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap",
                            "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.3)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    smi.terminate()
    lines = [l.split(",") for l in smi.communicate()[0].splitlines() if l.strip()]
    clk = [float(l[0]) for l in lines[3:-1]]
    pw = [float(l[1]) for l in lines[3:-1]]
    out[name] = {"ms": e0.elapsed_time(e1) / reps, "sm_mhz_median": statistics.median(clk) if clk else None,
                 "power_w_median": statistics.median(pw) if pw else None,
                 "power_cap_active": sum(1 for l in lines if "Active" in l[2]) / max(len(lines), 1)}
    print(name, out[name], flush=True)
print(json.dumps(out))
