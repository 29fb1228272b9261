"""Host-side multi-GPU logic on CPU: unit sharding, input slicing, the optional cache
gather and the max-over-ranks timing reduction, with world_size 2 over gloo."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2412_08521_b200.shard import gather_caches, slice_inputs, unit_shard


@pytest.mark.parametrize("B,Hkv,world", [(1, 8, 1), (1, 8, 2), (1, 8, 8), (4, 32, 8), (32, 8, 8),
                                         (3, 2, 4), (1, 3, 2), (5, 1, 3)])
def test_shards_partition_units(B, Hkv, world):
    seen = []
    for r in range(world):
        s = unit_shard(B, Hkv, world, r)
        seen.extend(range(s.unit_begin, s.unit_end))
    assert sorted(seen) == list(range(B * Hkv)) and len(seen) == len(set(seen))
    sizes = [unit_shard(B, Hkv, world, r).n_units for r in range(world)]
    assert max(sizes) - min(sizes) <= 1


def test_slice_inputs_views():
    B, Hkv, G, L, d = 2, 4, 2, 8, 4
    q = torch.arange(B * Hkv * G * L * d, dtype=torch.float32).reshape(B, Hkv * G, L, d)
    k = torch.arange(B * Hkv * L * d, dtype=torch.float32).reshape(B, Hkv, L, d)
    s = unit_shard(B, Hkv, 3, 1)  # units 3..5 -> (b0,h3), (b1,h0), (b1,h1)
    qs, ks, kw, vs = slice_inputs(q, k, k, k, s)
    assert ks.shape == (1, 3, L, d) and qs.shape == (1, 3 * G, L, d)
    assert torch.equal(ks[0, 0], k[0, 3]) and torch.equal(ks[0, 1], k[1, 0])
    assert torch.equal(qs[0, 2], q[1, 0])
    s1 = unit_shard(1, Hkv, 2, 1)
    qs, ks, _, _ = slice_inputs(q[:1], k[:1], k[:1], k[:1], s1)
    assert torch.equal(ks[0], k[0, 2:4]) and torch.equal(qs[0], q[0, 4:8])


def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _worker(rank, world, port, B, Hkv, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s = unit_shard(B, Hkv, world, rank)
        cache = {"lut_pos": torch.arange(s.unit_begin, s.unit_end, dtype=torch.int32)[:, None].repeat(1, 5),
                 "center_norm": torch.full((s.n_units, 3), float(rank))}
        full = gather_caches(cache, s, B * Hkv)
        t = torch.tensor([10.0 * (rank + 1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)  # bench.py: max over ranks
        q.put((rank, full["lut_pos"][:, 0].tolist(), full["center_norm"][:, 0].tolist(), t.item()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("B,Hkv", [(1, 8), (3, 1)])
def test_gloo_world2_gather_and_max(B, Hkv):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, B, Hkv, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, units, owners, tmax in res:
        assert units == list(range(B * Hkv))
        want = [float(r) for r in range(2) for _ in range(unit_shard(B, Hkv, 2, r).n_units)]
        assert owners == want
        assert tmax == 20.0
