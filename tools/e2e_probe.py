"""Where the end-to-end time of a decomposed march goes (run under torchrun):
upload of the host block, peer attach, the march, download -- rank 0 prints."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2211_16718_b200 as hd  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
os.environ.setdefault("TORCH_NCCL_HIGH_PRIORITY", "1")
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
spec = hd.GridSpec((512, 512, 512))
ic = hd.make_initial_condition(spec, hd.HitParams(), backend="torch")
lay = hd.decompose(spec, (1, 1, world))[rank]
state = hd.scatter(ic, [lay])[0]
del ic
torch.cuda.empty_cache()
halo = hd.DistHalo(lay)
gas = hd.GasModel(mu=0.006)
tp = hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=10)
halo.advance(state, gas, hd.TimeParams(scheme="rk4", cfl=0.4, max_steps=2), hd.DEFAULT_PARAMS, 0.0, 0.0,
             None, None, None)
host = torch.empty(state.data.numel(), dtype=torch.float64, pin_memory=True)
host.copy_(state.data)
out = torch.empty_like(host, pin_memory=True)
for rep in range(2):
    dist.barrier(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev = host.to("cuda", non_blocking=False)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    fs = hd.FieldSet(lay.spec, hd.Layout.COMPONENT_CONTIGUOUS, dev)
    r = halo.advance(fs, gas, tp, hd.DEFAULT_PARAMS, 0.0, 0.0, None, None, None)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    out.copy_(r.fields.data)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    v = torch.tensor([t1 - t0, t2 - t1, t3 - t2, t3 - t0], dtype=torch.float64, device="cuda")
    dist.all_reduce(v, op=dist.ReduceOp.MAX)
    if rank == 0:
        a = (1e3 * v).tolist()
        print(f"rep {rep} (max over ranks): upload {a[0]:.1f} ms, march {a[1]:.1f} ms, "
              f"download {a[2]:.1f} ms, total {a[3]:.1f} ms", flush=True)
dist.destroy_process_group()
