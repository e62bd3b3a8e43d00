"""Host-side multi-rank logic on CPU with the gloo backend (world size 2, 4 and 8 —
the (1, 1, 8) z slabs bench.py uses on 8 GPUs).

The NCCL path on the GPU uses exactly this code (DistHalo) on CUDA tensors;
here the z-slab halo protocol is checked against the monolithic periodic
fill, the way the reference checks RankHalo against a wrap-around slice
(pkg/tests/test_decomp.py:112-171).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2211_16718_b200 as hd


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _global_field(n, seed=3):
    rng = np.random.default_rng(seed)
    spec = hd.GridSpec(n)
    body = rng.standard_normal((5,) + spec.interior_shape)
    return spec, body


def _wrapped(spec, body):
    """Monolithic reference: ghosts filled by the periodic wrap x -> y -> z (grid.py:236-251)."""
    g = spec.ghost_width
    full = np.zeros((5,) + spec.shape)
    full[:, g:-g, g:-g, g:-g] = body
    for axis, nn in ((3, spec.n[0]), (2, spec.n[1]), (1, spec.n[2])):
        idx_lo = [slice(None)] * 4
        idx_src = [slice(None)] * 4
        idx_lo[axis], idx_src[axis] = slice(0, g), slice(nn, nn + g)
        full[tuple(idx_lo)] = full[tuple(idx_src)]
        idx_hi = [slice(None)] * 4
        idx_src2 = [slice(None)] * 4
        idx_hi[axis], idx_src2[axis] = slice(nn + g, nn + 2 * g), slice(g, 2 * g)
        full[tuple(idx_hi)] = full[tuple(idx_src2)]
    return full


def _worker(rank, world, port, n, q, dims):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        spec, body = _global_field(n)
        lay = hd.decompose(spec, dims)[rank]
        gfs = hd.FieldSet(spec, hd.Layout.COMPONENT_CONTIGUOUS,
                          torch.zeros(5 * spec.total_points, dtype=torch.float64))
        gfs.interior().copy_(torch.from_numpy(body))
        local = hd.scatter(gfs, [lay])[0]
        halo = hd.DistHalo(lay)
        halo.sync_fields(local)
        # expected: the monolithic wrapped field, cut to this rank's ghosted block
        full = _wrapped(spec, body)
        ox, oy, oz = lay.offset
        lx, ly, lz = lay.local_n
        g = spec.ghost_width
        # the wrapped global field is periodic, so the ghosted block is a periodic slice
        zs = np.arange(oz - g, oz + lz + g) % spec.n[2] + g
        ys = np.arange(oy - g, oy + ly + g) % spec.n[1] + g
        xs = np.arange(ox - g, ox + lx + g) % spec.n[0] + g
        want = full[:, zs][:, :, ys][:, :, :, xs]
        got = local.component_view().numpy()
        ok_fields = np.array_equal(got, want)
        # sync_scalars on one ghosted scalar (viscous.py:118 usage)
        arr = torch.zeros(lay.spec.shape, dtype=torch.float64)
        arr[g:-g, g:-g, g:-g] = torch.from_numpy(body[4, oz: oz + lz, oy: oy + ly, ox: ox + lx])
        halo.sync_scalars([arr], lay.spec.n, g)
        ok_scalar = np.array_equal(arr.numpy(), want[4])
        # a reduction like the dt provider: MAX is exact on every rank
        sig = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(sig, op=dist.ReduceOp.MAX)
        q.put((rank, ok_fields, ok_scalar, float(sig.item())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dims", [(1, 1, 2), (1, 1, 4), (2, 1, 1), (1, 2, 1), (2, 2, 1), (1, 2, 2),
                                  (2, 1, 2), (1, 1, 8)])
def test_block_halo_matches_monolithic_wrap(dims):
    """Every 3D block decomposition (decomp.py:66-103): after sync_fields each
    rank's ghosted block, edges and corners included, equals the periodic
    slice of the monolithically wrapped field."""
    world = dims[0] * dims[1] * dims[2]
    n = (4 * dims[0] + 2, 4 * dims[1] + 1, 4 * dims[2])
    n = tuple(n[d] if dims[d] == 1 else 4 * dims[d] for d in range(3))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q, dims)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_fields, ok_scalar, sig in results:
        assert ok_fields, f"rank {rank}: state ghosts differ from the periodic wrap"
        assert ok_scalar, f"rank {rank}: scalar ghosts differ from the periodic wrap"
        assert sig == float(world)


def test_decompose_and_numbering():
    spec = hd.GridSpec((16, 16, 32))
    lays = hd.decompose(spec, (1, 1, 4))
    assert [l.offset for l in lays] == [(0, 0, 0), (0, 0, 8), (0, 0, 16), (0, 0, 24)]
    assert lays[0].neighbor(2, -1) == 3 and lays[3].neighbor(2, +1) == 0
    assert hd.rank_of((1, 0, 2), (2, 2, 3)) == 1 + 2 * (0 + 2 * 2)
    assert hd.coords_of(9, (2, 2, 3)) == (1, 0, 2)
    # the reference's choice (pkg/tests/test_decomp.py:55-69): least face area, ties to x
    n = (16, 16, 16)
    assert hd.default_dims(1, n) == (1, 1, 1)
    assert hd.default_dims(2, n) == (2, 1, 1)
    assert hd.default_dims(4, n) == (4, 1, 1)
    assert hd.default_dims(8, n) == (4, 2, 1)
    assert hd.default_dims(8, (16, 16, 16), 3) == (4, 2, 1)
    with pytest.raises(hd.ConfigError):
        hd.default_dims(7, (16, 16, 16))  # 7 divides no extent
    # the drivers' GPU default: z slabs when legal, else the reference's choice
    assert hd.gpu_dims(8, (512, 512, 512)) == (1, 1, 8)
    assert hd.gpu_dims(4, (64, 64, 8)) == (4, 1, 1)  # local z extent 2 < ghost width
    assert hd.gpu_dims(8, (16, 16, 16)) == (4, 2, 1)
    with pytest.raises(hd.ConfigError):
        hd.decompose(spec, (1, 1, 3))
    with pytest.raises(hd.ConfigError):
        hd.decompose(hd.GridSpec((8, 8, 8)), (1, 1, 4))  # local 2 < ghost width 3


def test_scatter_gather_roundtrip():
    spec, body = _global_field((8, 6, 12))
    gfs = hd.FieldSet(spec, hd.Layout.COMPONENT_CONTIGUOUS,
                      torch.zeros(5 * spec.total_points, dtype=torch.float64))
    gfs.interior().copy_(torch.from_numpy(body))
    lays = hd.decompose(spec, (1, 1, 3))
    back = hd.gather(hd.scatter(gfs, lays), lays, spec)
    assert torch.equal(back.interior(), gfs.interior())
