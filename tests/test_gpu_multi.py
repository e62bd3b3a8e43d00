"""Decomposed runs on real GPUs (NCCL over NVLink), launched with torchrun from the test.

Needs >= 2 visible GPUs; skipped otherwise.  2- and (if available) 4-rank
runs of config 1 (32^3 HIT, RK4, CFL 0.4, mu 0.006) over every block shape
(z slabs, x and y splits, 2D splits) must equal the single-GPU run
bit-for-bit in exact mode (the reference's invariant,
pkg/tests/test_decomp.py:194-204) and to 1e-10 relative L2 in fast mode.
"""

import json
import os
import subprocess
import sys

import pytest
import torch

from conftest import ROOT

pytestmark = pytest.mark.gpu

SCRIPT = r'''
import hashlib, json, os, sys
sys.path.insert(0, os.environ["HD_ROOT"])
import numpy as np, torch, torch.distributed as dist
import paper_2211_16718_b200 as hd
rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
mode = os.environ["HD_TEST_MODE"]
spec = hd.GridSpec((32, 32, 32))
ic = hd.make_initial_condition(spec, hd.HitParams(), backend="numpy")
for dims in json.loads(os.environ["HD_TEST_DIMS"]):
    res = hd.parallel_advance(ic, hd.GasModel(mu=0.006), hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=10),
                              dims=tuple(dims), mode=mode)
    fin = res.fields.interior().cpu().numpy()
    if rank == 0:
        print("RESULT " + json.dumps({"dims": dims, "sha": hashlib.sha256(fin.tobytes()).hexdigest(),
                                      "t": res.t, "l2": [float(np.sqrt((fin[v] ** 2).sum())) for v in range(5)],
                                      "reports": [[r.rank, r.wall_seconds, r.comp_seconds, r.comm_seconds]
                                                  for r in res.reports]}))
# per-step records of the block march (z slabs): KE and enstrophy summed over ranks
lay = hd.decompose(spec, (1, 1, world))[rank]
local = hd.scatter(ic, [lay])[0]
res = hd.DistHalo(lay).advance(local, hd.GasModel(mu=0.006), hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=10),
                               hd.DEFAULT_PARAMS, 0.0, 0.0, None, None, mode)
if rank == 0:
    print("RECORDS " + json.dumps({"ke": [r.kinetic_energy for r in res.records],
                                   "enstrophy": [r.enstrophy for r in res.records]}))
dist.destroy_process_group()
'''


DIMS = {2: [(1, 1, 2), (2, 1, 1), (1, 2, 1)], 4: [(1, 1, 4), (2, 2, 1), (1, 2, 2), (2, 1, 2)]}


def _run(world, mode, tmp_path, dims=None, peer="1"):
    path = tmp_path / "pa.py"
    path.write_text(SCRIPT)
    dims = DIMS[world] if dims is None else dims
    env = dict(os.environ, HD_ROOT=ROOT, HD_TEST_MODE=mode, HD_TEST_DIMS=json.dumps(dims), HD_PEER=peer)
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          f"--nproc-per-node={world}", "--master-addr=127.0.0.1",
                          "--master-port=29533", str(path)], env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    res = [json.loads(l[7:]) for l in out.stdout.splitlines() if l.startswith("RESULT ")]
    assert [tuple(r["dims"]) for r in res] == [tuple(d) for d in dims]
    recs = [json.loads(l[8:]) for l in out.stdout.splitlines() if l.startswith("RECORDS ")]
    assert len(recs) == 1
    return res, recs[0]


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_decomposed_equals_single_gpu(tmp_path, traj32_golden, mode):
    ngpu = torch.cuda.device_count()
    if ngpu < 2:
        pytest.skip("needs >= 2 GPUs")
    import numpy as np

    for world in [w for w in (2, 4) if w <= ngpu]:
        res, recs = _run(world, mode, tmp_path)
        # diagnostics of the decomposed march: KE curve and enstrophy (combined over ranks)
        assert np.allclose(recs["ke"], traj32_golden["ke"][1:], rtol=1e-11, atol=0)
        assert np.allclose(recs["enstrophy"], traj32_golden["enstrophy"][1:], rtol=1e-11, atol=0)
        for r in res:
            # one TimingReport per rank; comm = exposed halo/collective waits (> 0: every
            # step waits for the dt reduction), comp = wall - comm
            assert [q[0] for q in r["reports"]] == list(range(world))
            for _, wall, comp, comm in r["reports"]:
                assert 0.0 < comm < wall and abs(comp + comm - wall) <= 1e-9 * wall
            if mode == "exact":
                assert r["sha"] == traj32_golden["final_sha256"], r["dims"]
                assert r["t"] == traj32_golden["t"]
            else:
                l2 = np.array(r["l2"])
                want = np.array(traj32_golden["l2"])
                assert np.all(np.abs(l2 - want) / want <= 1e-10), r["dims"]


def test_z_slab_nccl_halo_equals_single_gpu(tmp_path, traj32_golden):
    """z slabs default to the NVLink peer-store halo (hd_peer_*); HD_PEER=0 keeps
    the NCCL face exchange -- both must equal the single-GPU run bitwise."""
    ngpu = torch.cuda.device_count()
    if ngpu < 2:
        pytest.skip("needs >= 2 GPUs")
    world = 4 if ngpu >= 4 else 2
    res, recs = _run(world, "exact", tmp_path, dims=[(1, 1, world)], peer="0")
    for r in res:
        assert r["sha"] == traj32_golden["final_sha256"], r["dims"]
    import numpy as np

    assert np.allclose(recs["enstrophy"], traj32_golden["enstrophy"][1:], rtol=1e-11, atol=0)


TF_SCRIPT = r'''
import json, os, sys
sys.path.insert(0, os.environ["HD_ROOT"])
import torch, torch.distributed as dist
import paper_2211_16718_b200 as hd
rank = int(os.environ["RANK"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
spec = hd.GridSpec((32, 32, 32))
ic = hd.make_initial_condition(spec, hd.HitParams(), backend="numpy")
res = hd.parallel_advance(ic, hd.GasModel(mu=0.006), hd.TimeParams(scheme="rk4", cfl=0.4, t_final=0.2),
                          mode="exact")
if rank == 0:
    with open(os.path.join(os.environ["HD_OUT"], "tf.json"), "w") as fh:
        json.dump({"t": res.t, "steps": res.reports[0].steps,
                   "data": res.fields.interior().cpu().numpy().tobytes().hex()[:4096]}, fh)
dist.destroy_process_group()
'''


def test_t_final_march_on_two_gpus(tmp_path):
    """The host-synchronised march (t_final clipping, timeint.py:222-227) through the
    peer-store halo lands on t_final exactly and equals the single-GPU march."""
    ngpu = torch.cuda.device_count()
    if ngpu < 2:
        pytest.skip("needs >= 2 GPUs")
    import paper_2211_16718_b200 as hd

    path = tmp_path / "tf.py"
    path.write_text(TF_SCRIPT)
    env = dict(os.environ, HD_ROOT=ROOT, HD_OUT=str(tmp_path))
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node=2", "--master-addr=127.0.0.1", "--master-port=29545",
                          str(path)], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    with open(tmp_path / "tf.json") as fh:
        multi = json.load(fh)
    spec = hd.GridSpec((32, 32, 32))
    ic = hd.make_initial_condition(spec, hd.HitParams(), backend="numpy")
    res = hd.advance(ic, hd.GasModel(mu=0.006), hd.TimeParams(scheme="rk4", cfl=0.4, t_final=0.2),
                     mode="exact")
    assert res.t == multi["t"] == 0.2 and res.steps == multi["steps"]
    assert res.fields.interior().cpu().numpy().tobytes().hex()[:4096] == multi["data"]


def test_cli_scale_relaunches_one_process_per_gpu():
    """``scale`` outside torchrun relaunches itself with one rank per GPU and
    prints the reference's table (decomp.py:464-476) for each rank count."""
    ngpu = torch.cuda.device_count()
    if ngpu < 2:
        pytest.skip("needs >= 2 GPUs")
    out = subprocess.run([sys.executable, "-m", "paper_2211_16718_b200", "scale", "--ranks", "1,2",
                          "--steps", "2", "--set", "n=32", "--set", "scheme=rk4", "--port", "29547"],
                         cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    i = lines.index("ranks dims wall comp comm ratio speedup efficiency")
    rows = [l.split() for l in lines[i + 1:i + 3]]
    assert [r[0] for r in rows] == ["1", "2"] and rows[1][1] == "1x1x2"
    assert all(float(r[2]) > 0.0 for r in rows)


ERR_SCRIPT = r'''
import json, os, sys
sys.path.insert(0, os.environ["HD_ROOT"])
import numpy as np, torch, torch.distributed as dist
import paper_2211_16718_b200 as hd
rank = int(os.environ["RANK"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
n = 16
spec = hd.GridSpec((n, n, n))
fs = hd.FieldSet.zeros(spec, device="cpu")
it = fs.interior()
it[0] = 1.0
it[4] = 2.5
it[4, 13, 5, 6] = -1.0   # negative energy in the top z slab only
out = {}
for peer in ("1", "0"):
    os.environ["HD_PEER"] = peer
    try:
        hd.parallel_advance(fs, hd.GasModel(), hd.TimeParams(scheme="rk4", dt=0.01, max_steps=3))
        out[peer] = None
    except hd.StepError as e:
        out[peer] = [e.step, e.stage]
with open(os.path.join(os.environ["HD_OUT"], f"rank{rank}.json"), "w") as fh:
    json.dump({"rank": rank, "err": out}, fh)
dist.destroy_process_group()
'''


def test_step_error_raised_on_every_rank(tmp_path):
    """An invalid state in one rank's block: every rank raises the same StepError
    (error keys combined with MIN over ranks), none hangs in a collective."""
    ngpu = torch.cuda.device_count()
    if ngpu < 2:
        pytest.skip("needs >= 2 GPUs")
    path = tmp_path / "err.py"
    path.write_text(ERR_SCRIPT)
    env = dict(os.environ, HD_ROOT=ROOT, HD_OUT=str(tmp_path))
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node=2", "--master-addr=127.0.0.1", "--master-port=29541",
                          str(path)], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    res = []
    for r in range(2):
        with open(tmp_path / f"rank{r}.json") as fh:
            res.append(json.load(fh))
    assert len(res) == 2
    for r in res:
        assert r["err"]["1"] == [1, 0] and r["err"]["0"] == [1, 0], r


FULL_SCRIPT = r'''
import hashlib, json, os, sys
sys.path.insert(0, os.environ["HD_ROOT"])
import torch, torch.distributed as dist
import paper_2211_16718_b200 as hd
rank = int(os.environ["RANK"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
spec = hd.GridSpec((512, 512, 512))
ic = hd.make_initial_condition(spec, hd.HitParams(), backend="torch")
res = hd.parallel_advance(ic, hd.GasModel(mu=0.006), hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=2),
                          mode="exact")
if rank == 0:
    body = res.fields.interior().contiguous().cpu().numpy()
    with open(os.path.join(os.environ["HD_OUT"], "full.json"), "w") as fh:
        json.dump({"sha": hashlib.sha256(body.tobytes()).hexdigest(), "t": res.t}, fh)
dist.destroy_process_group()
'''


def test_512_z_slabs_equal_single_gpu_bitwise(tmp_path):
    """At the benchmark size (512^3, 2 RK4 steps, exact arithmetic) the 2-GPU z-slab
    run with the NVLink peer-store halo equals the single-GPU run bit-for-bit."""
    import hashlib

    ngpu = torch.cuda.device_count()
    if ngpu < 2:
        pytest.skip("needs >= 2 GPUs")
    import paper_2211_16718_b200 as hd

    path = tmp_path / "full.py"
    path.write_text(FULL_SCRIPT)
    env = dict(os.environ, HD_ROOT=ROOT, HD_OUT=str(tmp_path))
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node=2", "--master-addr=127.0.0.1", "--master-port=29543",
                          str(path)], env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    with open(tmp_path / "full.json") as fh:
        multi = json.load(fh)
    spec = hd.GridSpec((512, 512, 512))
    ic = hd.make_initial_condition(spec, hd.HitParams(), backend="torch", device="cuda:0")
    res = hd.advance(ic, hd.GasModel(mu=0.006), hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=2),
                     mode="exact")
    body = res.fields.interior().contiguous().cpu().numpy()
    hd.release_plans()
    assert hashlib.sha256(body.tobytes()).hexdigest() == multi["sha"]
    assert res.t == multi["t"]


HX_SCRIPT = r'''
import json, os, sys, ctypes
sys.path.insert(0, os.environ["HD_ROOT"])
import numpy as np, torch, torch.distributed as dist
import paper_2211_16718_b200 as hd
from paper_2211_16718_b200 import _lib
from paper_2211_16718_b200.decomp import _PeerLink
rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
dims = tuple(json.loads(os.environ["HD_DIMS"]))
spec = hd.GridSpec((16, 16, 16))
lay = hd.decompose(spec, dims)[rank]
halo = hd.DistHalo(lay)
plan = hd.get_plan(lay.spec, hd.GasModel(), periodic=halo.periodic)
assert _PeerLink.get(halo).attach(plan)
state = plan.fields(_lib.HD_BUF_STATE, 5)
# global field with known values: f(var, z, y, x) = var*1e6 + zg*1e4 + yg*1e2 + xg
g = spec.ghost_width
ln = lay.local_n
v = state.view((5,) + lay.spec.shape)
v.zero_()
z = torch.arange(ln[2], device="cuda")[:, None, None] + lay.offset[2]
y = torch.arange(ln[1], device="cuda")[None, :, None] + lay.offset[1]
x = torch.arange(ln[0], device="cuda")[None, None, :] + lay.offset[0]
for c in range(5):
    v[c, g:-g, g:-g, g:-g] = (c * 1e6 + z * 1e4 + y * 1e2 + x).double()
torch.cuda.synchronize(); dist.barrier()
L = _lib.load()
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
assert L.hd_halo_exchange(plan.h, ctypes.c_void_p(state.data_ptr()), 5, s) == 0
torch.cuda.synchronize(); dist.barrier()
# every face ghost (interior extent of the other axes) holds the periodic neighbour's value
ok = True
for d in range(3):
    for side in (0, 1):
        ax = 2 - d
        idx = list(range(0, g)) if side == 0 else list(range(ln[d] + g, ln[d] + 2 * g))
        got = v[0].index_select(ax, torch.tensor(idx, device="cuda"))
        got = got[tuple(slice(g, g + ln[2 - a]) if a != ax else slice(None) for a in range(3))]
        coord = torch.tensor([(lay.offset[d] + i - g) % spec.n[d] for i in idx], device="cuda").double()
        zz = (torch.arange(ln[2], device="cuda") + lay.offset[2]).double()
        yy = (torch.arange(ln[1], device="cuda") + lay.offset[1]).double()
        xx = (torch.arange(ln[0], device="cuda") + lay.offset[0]).double()
        comps = [zz, yy, xx]
        comps[ax] = coord
        want = comps[0][:, None, None] * 1e4 + comps[1][None, :, None] * 1e2 + comps[2][None, None, :]
        ok = ok and bool(torch.equal(got, want))
plan.peer_attach([None] * 3, [None] * 3)
with open(os.path.join(os.environ["HD_OUT"], f"hx{rank}.json"), "w") as fh:
    json.dump({"ok": ok}, fh)
dist.destroy_process_group()
'''


@pytest.mark.parametrize("dims", [(1, 1, 2), (2, 1, 1), (1, 2, 1)])
def test_halo_exchange_entry_point_peer(tmp_path, dims):
    """hd_halo_exchange on a peer-attached plan: every face ghost layer holds the
    neighbour's boundary layer (split axes) or the local wrap (periodic axes)."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    path = tmp_path / "hx.py"
    path.write_text(HX_SCRIPT)
    env = dict(os.environ, HD_ROOT=ROOT, HD_OUT=str(tmp_path), HD_DIMS=json.dumps(dims))
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node=2", "--master-addr=127.0.0.1", "--master-port=29547",
                          str(path)], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    for r in range(2):
        with open(tmp_path / f"hx{r}.json") as fh:
            assert json.load(fh)["ok"], r


RHS_SCRIPT = r'''
import hashlib, json, os, sys
sys.path.insert(0, os.environ["HD_ROOT"])
import numpy as np, torch, torch.distributed as dist
import paper_2211_16718_b200 as hd
rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
dims = tuple(json.loads(os.environ["HD_DIMS"]))
spec = hd.GridSpec((32, 32, 32))
ic = hd.make_initial_condition(spec, hd.HitParams(), backend="numpy")
gas = hd.GasModel(mu=0.006)
lay = hd.decompose(spec, dims)[rank]
local = hd.scatter(ic, [lay])[0]
halo = hd.DistHalo(lay)
inc = hd.make_rhs(gas, halo=halo, mode="exact")(local)
parts = [torch.empty_like(inc.interior().contiguous()) for _ in range(world)]
dist.all_gather(parts, inc.interior().contiguous())
if rank == 0:
    lays = hd.decompose(spec, dims)
    locs = []
    for r, part in enumerate(parts):
        fs = hd.FieldSet.zeros(lays[r].spec)
        fs.interior().copy_(part)
        locs.append(fs)
    glob = hd.gather(locs, lays, spec).interior().cpu().numpy()
    with open(os.path.join(os.environ["HD_OUT"], "rhs.json"), "w") as fh:
        json.dump({"sha": hashlib.sha256(np.ascontiguousarray(glob).tobytes()).hexdigest()}, fh)
dist.destroy_process_group()
'''


@pytest.mark.parametrize("dims", [(1, 1, 2), (2, 1, 1)])
def test_decomposed_make_rhs_equals_monolithic(tmp_path, dims):
    """make_rhs with a DistHalo (state faces, then the flux groups' faces between the
    viscous fluxes and their divergence: viscous.py:111-120) equals the single-GPU
    rhs bit-for-bit in exact mode."""
    import hashlib

    import numpy as np

    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    import paper_2211_16718_b200 as hd

    path = tmp_path / "rhs.py"
    path.write_text(RHS_SCRIPT)
    env = dict(os.environ, HD_ROOT=ROOT, HD_OUT=str(tmp_path), HD_DIMS=json.dumps(dims))
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node=2", "--master-addr=127.0.0.1", "--master-port=29549",
                          str(path)], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    with open(tmp_path / "rhs.json") as fh:
        multi = json.load(fh)
    spec = hd.GridSpec((32, 32, 32))
    ic = hd.make_initial_condition(spec, hd.HitParams(), backend="numpy")
    inc = hd.make_rhs(hd.GasModel(mu=0.006), mode="exact")(ic)
    body = np.ascontiguousarray(inc.interior().cpu().numpy())
    assert hashlib.sha256(body.tobytes()).hexdigest() == multi["sha"]


RK3_SCRIPT = r'''
import hashlib, json, os, sys
sys.path.insert(0, os.environ["HD_ROOT"])
import numpy as np, torch, torch.distributed as dist
import paper_2211_16718_b200 as hd
rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
spec = hd.GridSpec((32, 32, 32))
ic = hd.make_initial_condition(spec, hd.HitParams(), backend="numpy")
tp = hd.TimeParams(scheme="rk3", cfl=0.4, max_steps=4)
gas = hd.GasModel(mu=0.006)
out = {}
for mode in ("exact", "fast"):
    fins = []
    for dims in ((1, 1, world), (world, 1, 1)):
        res = hd.parallel_advance(ic, gas, tp, dims=dims, mode=mode)
        fins.append(res.fields.interior().cpu().numpy())
    if rank == 0:
        ref = hd.advance(ic, gas, tp, mode=mode).fields.interior().cpu().numpy()
        rel = [float(max(np.sqrt(((f[v] - ref[v]) ** 2).sum() / (ref[v] ** 2).sum()) for v in range(5)))
               for f in fins]
        out[mode] = {"decomposed": [hashlib.sha256(f.tobytes()).hexdigest() for f in fins],
                     "single": hashlib.sha256(ref.tobytes()).hexdigest(), "rel_l2": rel}
if rank == 0:
    print("RESULT " + json.dumps(out))
dist.destroy_process_group()
'''


def test_rk3_decomposed_equals_single_gpu(tmp_path):
    """TVD-RK3 (timeint.py:168-178) through the decomposed march (3 stages per step
    around the halo seam): z slabs and x splits equal the single-GPU march bit for
    bit in exact mode and to 1e-10 relative L2 in fast mode (the contract of
    test_decomposed_equals_single_gpu)."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    path = tmp_path / "rk3.py"
    path.write_text(RK3_SCRIPT)
    env = dict(os.environ, HD_ROOT=ROOT)
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node=2", "--master-addr=127.0.0.1", "--master-port=29537",
                          str(path)], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    res = [json.loads(l[7:]) for l in out.stdout.splitlines() if l.startswith("RESULT ")]
    assert len(res) == 1
    r = res[0]["exact"]
    assert r["decomposed"] == [r["single"]] * 2
    assert max(res[0]["fast"]["rel_l2"]) <= 1e-10
