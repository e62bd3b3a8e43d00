"""One RK4 step of the BASELINE workload at full size on the host CPU, timed for
the record (profiles/): the unmodified reference (hitdns from baseline/_ref,
workers = host threads) and the C oracle port (OpenMP), each on its own copy of
the reference's n^3 HIT IC.  The default bench reference arm samples 128^3
instead (its whole run must fit in minutes); this shows the per-point rate
holds at the metric's grid.

    python tools/reference_at_size.py [n] > gpurun_out/ref512.json
"""

import json
import os
import resource
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/hd_numba_cache")

import numpy as np  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
threads = len(os.sched_getaffinity(0))
out = {"n": n, "host_threads": threads, "steps": 1, "scheme": "rk4", "cfl": 0.4, "mu": 0.006}

import hitdns  # noqa: E402

gas = hitdns.GasModel(mu=0.006)
one = hitdns.TimeParams(scheme="rk4", cfl=0.4, max_steps=1)
small = hitdns.make_initial_condition(hitdns.GridSpec((16, 16, 16)), hitdns.HitParams())
hitdns.advance(small, gas, one, workers=threads)  # numba JIT outside the timing
t0 = time.perf_counter()
ic = hitdns.make_initial_condition(hitdns.GridSpec((n, n, n)), hitdns.HitParams())
out["ic_seconds"] = time.perf_counter() - t0
body = np.ascontiguousarray(ic.interior())
t0 = time.perf_counter()
r = hitdns.advance(ic, gas, one, workers=threads)
el = time.perf_counter() - t0
out["reference"] = {"seconds_per_step": el, "pt_step_per_s": n ** 3 / el, "dt": r.records[0].dt,
                    "peak_rss_gb": resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6}
print(json.dumps(out), flush=True)
del r, ic

from oracle import oracle as O  # noqa: E402

O.set_num_threads(threads)
P = O.Problem(n=(n, n, n), mu=0.006)
U = O.from_interior(body, P)
del body
t0 = time.perf_counter()
dts = O.advance(U, P, 1, cfl=0.4)
el = time.perf_counter() - t0
out["port"] = {"seconds_per_step": el, "pt_step_per_s": n ** 3 / el, "dt": float(dts[0]),
               "threads": O.num_threads(),
               "peak_rss_gb": resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6}
print(json.dumps(out), flush=True)
