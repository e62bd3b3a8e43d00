"""The paper's largest grid, decomposed: 1024^3 as z slabs over the ranks of
one box (4 GPUs: 1024 x 1024 x 256 per GPU, ~96 GB of workspace + state each;
the BASELINE config runs it on 8), RK4 (CFL 0.3: see --cfl), fast mode, peer-store halo.

The initial condition is the HIT field of the BASELINE workload (HitParams
defaults), synthesised across the ranks (hit.make_initial_condition_slab: a
counter-based mode generator, the shell energies summed over ranks, a slab FFT
with one all-to-all), so no rank ever holds the global transform; its shell
spectrum is checked against the target.  --ic tg gives the smooth Taylor-Green
field of round 1 instead.  Checks: finite, global mass conserved, KE decays.

    torchrun --nproc-per-node 4 tools/big_decomp.py [--grid 1024] [--steps 100] [--warmup 3]
"""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2211_16718_b200 as hd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--grid", type=int, default=1024)
ap.add_argument("--nz", type=int, default=0, help="global z extent (default: --grid); e.g. "
                "512 x 512 x 256 on 4 GPUs gives each the 64-plane slab of 512^3 on 8")
ap.add_argument("--dims", default="", help="block shape x,y,z (default 1,1,world)")
ap.add_argument("--steps", type=int, default=100)
ap.add_argument("--warmup", type=int, default=3)
# The reference's dt is convective only (timeint.py:122-138).  With mu = 0.006 the
# 4th-order viscous/heat-conduction operator (D4 applied twice: |k* h|^2 <= 1.883 per
# axis; diffusivity gamma mu / Pr = 0.0117) is RK4-stable only for dt <= 2.785 h^2 /
# (3 * 1.883 * 0.0117) = 42 h^2: at 1024^3 that is 1.59e-3 while CFL 0.4 gives 1.8e-3,
# and the march stops with StepError (nonpositive pressure) after ~80 steps; CFL 0.3 is stable.
ap.add_argument("--cfl", type=float, default=0.3)
ap.add_argument("--ic", default="hit", choices=["hit", "tg"])
a = ap.parse_args()

rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
os.environ.setdefault("TORCH_NCCL_HIGH_PRIORITY", "1")
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
n = a.grid
nz = a.nz or n
spec = hd.GridSpec((n, n, nz), (2 * math.pi, 2 * math.pi, 2 * math.pi * nz / n))
dims = tuple(int(v) for v in a.dims.split(",")) if a.dims else (1, 1, world)
lay = hd.decompose(spec, dims)[rank]
spectrum_check = None
if a.ic == "hit":
    fs = hd.make_initial_condition_slab(spec, hd.HitParams(), lay)
    # the shell spectrum of the synthesised field (slab FFT, shells summed over ranks)
    # against the target on every populated shell above round-off
    it = fs.interior()
    table = hd.compute_spectrum_slab(*(it[1 + d] / it[0] for d in range(3)), lay.coords[2], dims[2])
    torch.cuda.empty_cache()
    want = hd.target_spectrum(np.arange(1, n // 2, dtype=np.float64))
    got = table.energy[1:n // 2]
    above = want > 1e-13
    spectrum_check = {"shells": int(above.sum()),
                      "max_rel_err": float(np.max(np.abs(got[above] - want[above]) / want[above])),
                      "ke": table.total()}
else:
    fs = hd.FieldSet.zeros(lay.spec)
    it = fs.interior()
h = 2 * math.pi / n
ox, oy, oz = lay.offset
ly = lay.local_n[1]
lx = lay.local_n[0]
lz = lay.local_n[2]
if a.ic == "tg":
    # one period over the z extent (the box is 2 pi nz / n long; the spacing stays h)
    z = (oz + torch.arange(lz, dtype=torch.float64, device="cuda"))[:, None, None] * (2 * math.pi / nz)
    y = (oy + torch.arange(ly, dtype=torch.float64, device="cuda"))[None, :, None] * h
    x = (ox + torch.arange(lx, dtype=torch.float64, device="cuda"))[None, None, :] * h
    # Taylor-Green-like velocity (divergence-free) plus a k = 4 perturbation, rho = 1, p = 1/gamma
    u0 = 0.3
    it[0] = 1.0
    it[1] = u0 * torch.sin(x) * torch.cos(y) * torch.cos(z) + 0.05 * torch.sin(4 * y) * torch.cos(4 * z)
    it[2] = -u0 * torch.cos(x) * torch.sin(y) * torch.cos(z) + 0.05 * torch.sin(4 * z) * torch.cos(4 * x)
    it[3] = 0.05 * torch.sin(4 * x) * torch.cos(4 * y)
    it[4] = (1.0 / 1.4) / 0.4 + 0.5 * (it[1] ** 2 + it[2] ** 2 + it[3] ** 2)
    del x, y, z
torch.cuda.empty_cache()
gas = hd.GasModel(mu=0.006)
halo = hd.DistHalo(lay)


def march(state, steps):
    tp = hd.TimeParams(scheme="rk4", cfl=a.cfl, max_steps=steps)
    return halo.advance(state, gas, tp, hd.DEFAULT_PARAMS, 0.0, 0.0, None, None, None)


def mass(state):
    t = state.interior()[0].sum().reshape(1) * lay.spec.cell_volume()
    dist.all_reduce(t)
    return float(t.item())


m0 = mass(fs)
res = march(fs, a.warmup)
res_first_ke = res.records[0].kinetic_energy
dist.barrier()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
res = march(res.fields, a.steps)
e1.record()
dist.barrier()
torch.cuda.synchronize()
ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
dist.all_reduce(ms, op=dist.ReduceOp.MAX)
ms = float(ms.item())
fin = torch.tensor([float(torch.isfinite(res.fields.interior()).all())], device="cuda")
dist.all_reduce(fin, op=dist.ReduceOp.MIN)
m1 = mass(res.fields)
peak = torch.tensor([torch.cuda.max_memory_allocated() / 1e9], dtype=torch.float64, device="cuda")
dist.all_reduce(peak, op=dist.ReduceOp.MAX)
if rank == 0:
    out = {"grid": [n, n, nz], "n_gpus": world, "dims": list(dims), "steps": a.steps, "cfl": a.cfl,
           "warmup": a.warmup, "ms_per_step": ms / a.steps,
           "pt_step_per_s": n * n * nz * a.steps / (ms / 1e3), "t": res.t,
           "finite": bool(fin.item() == 1.0), "mass_rel_change": abs(m1 - m0) / abs(m0),
           "peak_mem_gb_max_rank": float(peak.item()),
           "peer_halo": any(l.digests is not None for l in hd.decomp._PeerLink._cache.values()),
           "ic": a.ic, "ic_spectrum": spectrum_check,
           "ke_first": res_first_ke, "ke_last": res.records[-1].kinetic_energy,
           "enstrophy_last": res.records[-1].enstrophy}
    print(json.dumps(out))
dist.destroy_process_group()
