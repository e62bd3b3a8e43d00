"""Benchmark: grid-point RK4-step updates/s (fp64) of the HIT decay problem.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--n 512] [--mode fast|exact]
    python bench.py --impl reference ...        # the CPU reference arm (hitdns itself)

One step = what the reference's ``advance`` does per step (timeint.py:224-257):
CFL dt (global max reduction), one classical RK4 step (4 x [ghost sync,
WENO5/Roe hyperbolic RHS, 4th-order viscous RHS, stage update]) and the
step diagnostics (mass, momentum, energy, max wavespeed, KE).

N = 1: workload 512^3 (the metric's grid, BASELINE.json), HIT IC (HitParams
defaults, synthesised on the GPU), mu = 0.006, CFL 0.4.  N > 1 (torchrun, one
rank per GPU): the same 512^3 problem split along z (strong scaling), NCCL
halo exchange overlapped with the x/y sweeps.  Rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ALG_BYTES_PER_PT_STEP = 680.0      # compulsory SoA traffic of a fused RK4 step
ALG_FLOPS_PER_PT_STEP = 17.9e3 + 1550.0  # flops + div/sqrt counted as one
SWEEP_FLOPS_PER_PT = 1406.0 + 125.0 + 3.0 + 10.0  # per interface (K:97-204) + flux components
MU = 0.006
# Algorithmic (bytes, reference flops) per interior point and launch of each stage kernel
# (fast mode): the reference counts 1,406 flops + 125 div + 3 sqrt per interface
# + ~10 for the flux components; central differences 6 flops each.
_SW = SWEEP_FLOPS_PER_PT
KERNEL_COST = {
    "sweep_x": (80.0, _SW),                       # u 40 + inc 40 (overwrite)
    "sweep_y": (176.0, _SW + 8 * 7),              # u 40 + inc RMW 80 + F_x, F_y (7 fields) 56
    # stage average: u 40 + inc 40 + F_z 32 + u_n 30 + acc 30 | out 40 + acc 30
    # (u_n and acc are not read at stage 1, acc not written at stage 4)
    "sweep_z": (242.0, _SW + 4 * 7 + 15 + 12),
    "gradflux": (112.0, 12 * 6 + 40 + 14),        # state 40 | 9 flux fields 72
    "prims": (72.0, 15.0),
    "divergence": (192.0, 12 * 7 + 15),           # exact mode: 9 fields + inc, u, acc | out, acc
    "reduce": (40.0, 30.0),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--grid", "--n", dest="n", type=int, default=512,
                    help="cube size (use --grid under torchrun: --n collides with its options)")
    ap.add_argument("--mode", default="fast", choices=["fast", "exact"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-n", type=int, default=128)
    ap.add_argument("--dims", default=None,
                    help="block decomposition px,py,pz for N>1 (default: z slabs 1,1,N)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
class ClockSampler:
    """Clocks + throttle reasons during the timed region: one `nvidia-smi -lms 200`
    process (the profiling recipe's clocks line), stopped by its own handle."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._proc = None

    def __enter__(self):
        try:
            self._proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                           "--format=csv,noheader,nounits", "-lms", "200"],
                                          stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:  # noqa: BLE001 - no nvidia-smi: reported as unsampled
            self._proc = None
        return self

    def __exit__(self, *exc):
        if self._proc is None:
            return
        self._proc.terminate()
        try:
            out, _ = self._proc.communicate(timeout=10)
        except subprocess.TimeoutExpired:
            self._proc.kill()
            out, _ = self._proc.communicate()
        for line in out.splitlines():
            if line.strip():
                self.samples.append([x.strip() for x in line.split(",")])

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower().startswith("active")})
        pw = [float(s[6]) for s in self.samples if len(s) > 6 and s[6].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples), "power_w": statistics.median(pw) if pw else None}


# ---------------------------------------------------------------------------
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def host_threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


def reference_cpu(n: int, steps: int, warmup: int, budget_s: float | None = None):
    """The unmodified reference package (hitdns 0.1.0 from baseline/_ref, numba
    kernels) through its public API: ``hitdns.advance(..., workers=<host threads>)``
    one RK4 step per call (CFL dt, stepper, diagnostics: timeint.py:199-258) on
    its own n^3 HIT IC.  None when the package (or numba) is not importable."""
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join("/tmp", "hd_numba_cache"))
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import hitdns
    except ImportError:
        return None
    workers = host_threads()
    ic = hitdns.make_initial_condition(hitdns.GridSpec((n, n, n)), hitdns.HitParams())
    gas = hitdns.GasModel(mu=MU)
    one = hitdns.TimeParams(scheme="rk4", cfl=0.4, max_steps=1)
    fields, t = ic, 0.0
    for _ in range(max(warmup, 1)):  # the first call also JIT-compiles the numba kernels
        r = hitdns.advance(fields, gas, one, workers=workers, t0=t)
        fields, t = r.fields, r.t
    t0 = time.perf_counter()
    done = 0
    while done < steps:
        r = hitdns.advance(fields, gas, one, workers=workers, t0=t)
        fields, t = r.fields, r.t
        done += 1
        if budget_s is not None and time.perf_counter() - t0 > budget_s:
            break
    el = time.perf_counter() - t0
    return n ** 3 * done / el, done, el, workers


def cpu_reference(n: int, steps: int, warmup: int, budget_s: float | None = None):
    """The C oracle port of the reference path (OpenMP, all host threads): the
    fallback CPU baseline when the reference package is not installed."""
    import numpy as np

    from oracle import oracle as O
    from paper_2211_16718_b200.hit import HitParams, synthesize_velocity

    O.lib()
    # every host thread, even under torchrun (which exports OMP_NUM_THREADS=1)
    O.set_num_threads(host_threads())
    u, v, w = synthesize_velocity(n, HitParams(), "numpy")
    body = np.empty((5, n, n, n))
    body[0] = 1.0
    body[1], body[2], body[3] = u, v, w
    body[4] = (1.0 / 1.4) / 0.4 + 0.5 * (u * u + v * v + w * w)
    P = O.Problem(n=(n, n, n), mu=MU)
    U = O.from_interior(body, P)
    for _ in range(warmup):
        O.advance(U, P, 1, cfl=0.4)
    t0 = time.perf_counter()
    done = 0
    while done < steps:
        O.advance(U, P, 1, cfl=0.4)
        done += 1
        if budget_s is not None and time.perf_counter() - t0 > budget_s and done >= 1:
            break
    el = time.perf_counter() - t0
    return n ** 3 * done / el, done, el, O.num_threads()


def metric_name(n: int) -> str:
    return f"grid-point RK4-step updates/sec (fp64, {n}^3)"


def workload_config(args, world: int, dims=None) -> dict:
    """The ``config`` object of both arms (the same workload)."""
    return {"workload": f"HIT decay {args.n}^3, WENO5+Roe, 4th-order viscous, RK4, CFL 0.4",
            "grid": args.n, "scheme": "rk4", "cfl": 0.4, "mu": MU, "mode": args.mode,
            "parallelism": f"blocks {'x'.join(map(str, dims))}" if world > 1 else "single GPU",
            "l2": "state 5.6 GB >> 126 MB L2 (no flush needed)",
            "ic": "HIT (HitParams defaults) synthesised on the GPU (torch backend)"}


def cpu_baseline(n: int, steps: int, warmup: int, budget_s: float, metric_n: int = 512):
    """(rate, steps done, seconds, threads, kind, sample text, config overrides):
    the reference package itself when installed (kind "reference"), else the C port."""
    got = reference_cpu(n, steps, warmup, budget_s)
    if got is not None:
        rate, done, el, threads = got
        return rate, done, el, threads, "reference", (
            f"hitdns 0.1.0 (the unmodified reference, baseline/_ref) hitdns.advance(..., "
            f"workers={threads}) on its own {n}^3 HIT IC, RK4 CFL 0.4 mu {MU}: {done} steps in "
            f"{el:.1f} s after {max(warmup, 1)} warm-up (numba JIT)"), {
                "grid": n, "parallelism": f"CPU, {threads} host threads (hitdns workers)",
                "ic": "hitdns.make_initial_condition (the reference's numpy synthesis)",
                "sample": f"per-point rate measured on {n}^3 (the cost per point is "
                          f"data-independent); the metric's grid is {metric_n}^3"}
    rate, done, el, threads = cpu_reference(n, steps, warmup, budget_s)
    return rate, done, el, threads, "port", (
        f"C oracle port (oracle/hd_oracle.c, OpenMP, {threads} threads) on a {n}^3 sample of the "
        f"same HIT RK4 problem: {done} steps in {el:.1f} s"), {
            "grid": n, "parallelism": f"CPU, {threads} OpenMP threads (C port of the reference)",
            "ic": "hit.py numpy synthesis",
            "sample": f"per-point rate measured on {n}^3; the metric's grid is {metric_n}^3"}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n = args.cpu_n
    rate, done, el, threads, kind, sample, cfg = cpu_baseline(n, args.steps, args.warmup, 150.0, args.n)
    config = dict(workload_config(args, 1))
    config.update(cfg)
    for key in ("mode", "l2"):  # GPU-arm settings that do not apply to a CPU run
        config.pop(key, None)
    line = {
        "metric": metric_name(args.n), "impl": "reference",
        "value": rate, "unit": "pt*step/s", "n_gpus": args.gpus, "steps": done,
        "warmup": args.warmup, "ms_per_step": 1e3 * el / done, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config,
        "cpu_baseline": {"value": rate, "unit": "pt*step/s", "cores": threads, "kind": kind,
                         "sample": sample},
        "e2e": {"value": rate, "unit": "pt*step/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def fp64_peak(hd, torch):
    """Measured DFMA throughput (TFLOP/s) of this GPU: hd_fp64_probe."""
    import ctypes

    L = hd._lib.load(require_cuda=True)
    sm = torch.cuda.get_device_properties(0).multi_processor_count
    blocks, threads, iters = sm * 8, 256, 4096
    out = torch.empty(blocks * threads, dtype=torch.float64, device="cuda")
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for _ in range(2):
        L.hd_fp64_probe(ctypes.c_void_p(out.data_ptr()), blocks, threads, iters, s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 5
    for _ in range(reps):
        L.hd_fp64_probe(ctypes.c_void_p(out.data_ptr()), blocks, threads, iters, s)
    e1.record()
    torch.cuda.synchronize()
    sec = e0.elapsed_time(e1) / 1e3 / reps
    return 2.0 * 8 * iters * threads * blocks / sec / 1e12


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
        return
    import torch
    import torch.distributed as dist

    import paper_2211_16718_b200 as hd

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        # NCCL's halo kernels on high-priority streams: their CTAs are scheduled ahead of
        # the waiting sweep blocks, so the exchange overlaps instead of queueing behind
        # (512^3 on 4 GPUs: 31.8 -> 31.1 ms/step)
        os.environ.setdefault("TORCH_NCCL_HIGH_PRIORITY", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n = args.n
    spec = hd.GridSpec((n, n, n))
    gas = hd.GasModel(mu=MU)
    hd.set_mode(args.mode)

    # ---- initial condition (identical on every rank; each keeps its z slab) --
    ic = hd.make_initial_condition(spec, hd.HitParams(), backend="torch")
    if world > 1:
        dims = tuple(int(x) for x in args.dims.split(",")) if args.dims else (1, 1, world)
        lay = hd.decompose(spec, dims)[rank]
        state = hd.scatter(ic, [lay])[0]
        halo = hd.DistHalo(lay)
    else:
        lay, state, halo = None, ic, None
    del ic
    torch.cuda.empty_cache()
    lspec = state.spec

    def march(fs, steps):
        tp = hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=steps)
        if halo is None:
            return hd.advance(fs, gas, tp)
        return halo.advance(fs, gas, tp, hd.DEFAULT_PARAMS, 0.0, 0.0, None, None, None)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- warm-up --------------------------------------------------------------
    res = march(state, args.warmup)
    state = res.fields
    barrier()

    # ---- timed region -------------------------------------------------------------
    L = hd._lib.load()
    plan = hd.get_plan(lspec, gas, periodic=halo.periodic if halo else (True, True, True))
    plan.timer_read()  # drop warm-up records
    plan.timer_enable(True)  # CUDA events around every stage kernel, on its stream
    launches0 = L.hd_launch_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        barrier()
        e0.record()
        res = march(state, args.steps)
        e1.record()
        barrier()
    launches = L.hd_launch_counter() - launches0
    ktimes = plan.timer_read()
    plan.timer_enable(False)
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    total_pts = n ** 3
    value = total_pts * args.steps / (ms / 1e3)
    recs = res.records
    state = res.fields

    # ---- roofline of the dominant kernel, timed inside the timed region ---------------
    peak_fp64 = fp64_peak(hd, torch)
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
        peaks = json.load(fh)
    hbm_peak = float(peaks["hbm_gbs"])
    lpts = lspec.interior_points
    kernels = {}
    for kind, (tot, cnt) in ktimes.items():
        if not cnt:
            continue
        avg = tot / cnt
        b, f = KERNEL_COST.get(kind, (0.0, 0.0))
        kernels[kind] = {"avg_ms": avg, "launches": cnt, "share": tot / ms,
                         "GB_s": lpts * b / (avg / 1e3) / 1e9,
                         "TFLOP_s": lpts * f / (avg / 1e3) / 1e12}
    top = max(kernels, key=lambda k: kernels[k]["avg_ms"] * kernels[k]["launches"])
    kt = kernels[top]
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "sweep_dram_bytes.json")
    if os.path.exists(tfile):
        with open(tfile) as fh:
            tr = json.load(fh)
        if tr.get("n") == n and world == 1 and tr.get("kernel") == top:
            traffic = tr.get("bytes_per_launch")
    roofline = {
        "bound": "hbm", "achieved": kt["GB_s"], "peak": hbm_peak, "unit": "GB/s",
        "frac": kt["GB_s"] / hbm_peak, "traffic": traffic, "kernel": top,
        "note": ("the stencil is FP64-pipe-bound: fp64.frac is the binding one; algorithmic "
                 "bytes/flops per point in KERNEL_COST (bench.py) and DESIGN.md sec. 3"),
        "fp64": {"achieved_tflops": kt["TFLOP_s"], "peak_tflops_measured": peak_fp64,
                 "frac": kt["TFLOP_s"] / peak_fp64},
        "step": {"hbm_frac": value / world * ALG_BYTES_PER_PT_STEP / (hbm_peak * 1e9),
                 "fp64_frac": value / world * ALG_FLOPS_PER_PT_STEP / (peak_fp64 * 1e12)},
        "kernels": kernels,
    }

    # ---- end-to-end through the public API with host buffers ------------------------
    e2e = None
    if not args.no_e2e:
        host_in = torch.empty(state.data.numel(), dtype=torch.float64, pin_memory=True)
        host_in.copy_(state.data)
        host_out = torch.empty_like(host_in, pin_memory=True)
        barrier()
        t0 = time.perf_counter()
        fs_host = hd.FieldSet(lspec, hd.Layout.COMPONENT_CONTIGUOUS, host_in)
        r2 = march(fs_host, args.steps)
        host_out.copy_(r2.fields.data, non_blocking=True)
        barrier()
        el = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([el], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        nbytes = host_in.numel() * 8
        e2e = {"value": total_pts * args.steps / el, "unit": "pt*step/s",
               "h2d_bytes_per_step": nbytes * world / args.steps,
               "d2h_bytes_per_step": (nbytes * world + 11 * 8 * args.steps) / args.steps,
               "how": "hd.advance(host pinned FieldSet) -> K steps -> final state to pinned host; "
                      "one upload + one download per K-step run, amortised per step"}

    # ---- CPU baseline (rank 0, N = 1 only) -----------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        rate, done, el, threads, kind, sample, _ = cpu_baseline(args.cpu_n, 100, 1, 15.0, n)
        cpu = {"value": rate, "unit": "pt*step/s", "cores": threads, "kind": kind, "sample": sample}

    if rank == 0:
        line = {
            "metric": metric_name(n),
            "value": value, "unit": "pt*step/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, world, lay.dims if world > 1 else None),
            "gpu_launches": int(launches),
            "clocks": clocks.summary(),
            "roofline": roofline,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "diagnostics": {"ke_first": recs[0].kinetic_energy, "ke_last": recs[-1].kinetic_energy,
                            "dt_last": recs[-1].dt, "mass": recs[-1].mass},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
