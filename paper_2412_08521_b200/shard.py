"""Multi-GPU partitioning of the prefill-compress path.

Units (one KV head of one sequence with its G query heads) share nothing, so the
path shards with no data-path collective: each rank compresses its own units.
The only optional collective is a gather of the fixed-size compressed caches
(NCCL over NVLink on B200, gloo in the CPU tests), off the timed path.

Sharding rule: contiguous blocks of KV heads when H_kv is divisible by the world
size (one KV head per GPU for configs 3 and 5 at 8 GPUs); otherwise contiguous
blocks of the flattened (b, h_kv) unit index, which degenerates to sharding by
batch when H_kv is small."""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    unit_begin: int   # flattened unit index u = b * H_kv + h_kv, [begin, end)
    unit_end: int
    by_head: bool     # True: same batch rows, a head slice [h0, h1) of every sequence

    @property
    def n_units(self) -> int:
        return self.unit_end - self.unit_begin


def unit_shard(batch: int, heads_kv: int, world: int, rank: int) -> Shard:
    if world <= 0 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    if batch == 1 and heads_kv % world == 0:
        per = heads_kv // world
        return Shard(rank, world, rank * per, (rank + 1) * per, True)
    total = batch * heads_kv
    base, extra = divmod(total, world)
    begin = rank * base + min(rank, extra)
    end = begin + base + (1 if rank < extra else 0)
    return Shard(rank, world, begin, end, False)


def slice_inputs(q_rot, k_rot, k_raw, v, shard: Shard):
    """Views of [B, H, L, d] tensors holding only the shard's units.

    by_head shards (B == 1) are zero-copy head slices; unit-range shards gather rows
    of the flattened [(B*H_kv), ...] layout (contiguous when the range is)."""
    B, Hq, L, d = q_rot.shape
    Hkv = k_rot.shape[1]
    G = Hq // Hkv
    if shard.by_head:
        h0, h1 = shard.unit_begin, shard.unit_end
        return (q_rot[:, h0 * G:h1 * G], k_rot[:, h0:h1], k_raw[:, h0:h1], v[:, h0:h1])
    u0, u1 = shard.unit_begin, shard.unit_end
    qf = q_rot.reshape(B * Hkv, G, L, d)[u0:u1].reshape(1, (u1 - u0) * G, L, d)
    kf = k_rot.reshape(B * Hkv, L, d)[u0:u1].reshape(1, u1 - u0, L, d)
    kw = k_raw.reshape(B * Hkv, L, d)[u0:u1].reshape(1, u1 - u0, L, d)
    vf = v.reshape(B * Hkv, L, d)[u0:u1].reshape(1, u1 - u0, L, d)
    return qf, kf, kw, vf


def gather_caches(cache: dict, shard: Shard, total_units: int, group=None) -> dict:
    """All-gather each rank's fixed-size per-unit cache tensors into [total_units, ...].

    Every rank must hold the same per-unit capacities (equal budget per head,
    PAPER.md:323), so the gather is a plain all_gather of equal-sized blocks."""
    import torch
    import torch.distributed as dist

    world = shard.world
    sizes = [unit_shard_size(total_units, world, r) for r in range(world)]
    mx = max(sizes)
    out = {}
    for name, t in cache.items():
        pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[: t.shape[0]] = t
        parts = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad, group=group)
        out[name] = torch.cat([p[:s] for p, s in zip(parts, sizes)], dim=0)
    return out


def unit_shard_size(total_units: int, world: int, rank: int) -> int:
    base, extra = divmod(total_units, world)
    return base + (1 if rank < extra else 0)
