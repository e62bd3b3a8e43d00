"""The slab-decomposed HIT synthesis (hit.synthesize_velocity_slab, the IC of the
1024^3 configuration) on CPU with gloo ranks: every rank count gives the same
field (FFT round-off), and the field has the properties the reference pins for
its own synthesis (pkg/tests/test_hit.py:48-75): each populated shell carries
exactly the target spectrum, the field is solenoidal and real, KE ~ 3/2 u0^2."""

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


def _worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        u, v, w = hd.synthesize_velocity_slab(n, hd.HitParams(), rank, world, device="cpu")
        q.put((rank, u.numpy(), v.numpy(), w.numpy()))
    finally:
        dist.destroy_process_group()


def _slabs(n, world):
    if world == 1:
        return [tuple(t.numpy() for t in hd.synthesize_velocity_slab(n, hd.HitParams(), device="cpu"))]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, PORTS[world], n, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = dict((r, (u, v, w)) for r, u, v, w in (q.get(timeout=120) for _ in range(world)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return [got[r] for r in range(world)]


PORTS = {}


@pytest.fixture(scope="module")
def fields16():
    n = 16
    out = {}
    for world in (1, 2, 4):
        PORTS[world] = _free_port()
        slabs = _slabs(n, world)
        out[world] = tuple(np.concatenate([s[a] for s in slabs], axis=0) for a in range(3))
    return out


def test_slab_field_is_decomposition_invariant(fields16):
    ref = fields16[1]
    for world in (2, 4):
        for a in range(3):
            scale = np.abs(ref[a]).max()
            assert np.abs(fields16[world][a] - ref[a]).max() <= 1e-14 * scale


def test_slab_field_matches_the_target_spectrum(fields16):
    n = 16
    u, v, w = fields16[4]
    table = hd.compute_spectrum(u, v, w)
    want = hd.target_spectrum(np.arange(1, n // 2, dtype=np.float64))
    np.testing.assert_allclose(table.energy[1:n // 2], want, rtol=1e-12, atol=0.0)
    assert table.energy[0] < 1e-30 and np.all(table.energy[n // 2:] < 1e-20)
    assert hd.spectral_divergence(u, v, w) < 1e-12 * 0.3 * 4.0


def test_slab_field_kinetic_energy_and_seed():
    u, v, w = (t.numpy() for t in hd.synthesize_velocity_slab(32, hd.HitParams(), device="cpu"))
    ke = 0.5 * float(np.mean(u * u + v * v + w * w))
    assert ke == pytest.approx(0.135, rel=0.05)
    u2 = hd.synthesize_velocity_slab(32, hd.HitParams(seed=7), device="cpu")[0].numpy()
    assert not np.array_equal(u, u2)
    again = hd.synthesize_velocity_slab(32, hd.HitParams(), device="cpu")[0].numpy()
    assert np.array_equal(u, again)


def test_slab_initial_condition_block():
    spec = hd.GridSpec((16, 16, 16))
    lay = hd.decompose(spec, (1, 1, 1))[0]
    fs = hd.make_initial_condition_slab(spec, hd.HitParams(), lay, device="cpu")
    it = fs.interior()
    assert bool((it[0] == 1.0).all())
    v2 = (it[1] ** 2 + it[2] ** 2 + it[3] ** 2) / it[0] ** 2
    p = 0.4 * (it[4] - 0.5 * it[0] * v2)
    assert torch.allclose(p, torch.full_like(p, 1.0 / 1.4), rtol=1e-12, atol=0)
    with pytest.raises(hd.ConfigError):
        hd.make_initial_condition_slab(spec, hd.HitParams(), hd.decompose(spec, (2, 1, 1))[0], device="cpu")


def _spec_worker(rank, world, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        u, v, w = hd.synthesize_velocity_slab(n, hd.HitParams(), rank, world, device="cpu")
        table = hd.compute_spectrum_slab(u, v, w, rank, world)
        q.put((rank, table.energy))
    finally:
        dist.destroy_process_group()


def test_slab_spectrum_matches_the_global_one():
    """compute_spectrum_slab over 4 gloo ranks equals compute_spectrum of the whole field."""
    n, world = 16, 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_spec_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    tables = [q.get(timeout=120)[1] for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    u, v, w = (t.numpy() for t in hd.synthesize_velocity_slab(n, hd.HitParams(), device="cpu"))
    want = hd.compute_spectrum(u, v, w).energy
    for got in tables:
        np.testing.assert_allclose(got[: len(want)], want[: len(got)], rtol=1e-12, atol=1e-30)
