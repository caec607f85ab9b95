"""Multi-GPU plumbing: one process per GPU, engine shards, one counter all-reduce.

SURVEY §8(e): shard r of N owns engines [r*P/N, (r+1)*P/N) and a 1/N slice of
the global unit; it regenerates its halo and the global points from the seeds,
so the only exchange is the final sum of (edges, fingerprint, comps) — exact in
any order because the fingerprint is a wrapping u64 sum.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

U64 = 1 << 64


def _to_i64(x: int) -> int:
    x %= U64
    return x - U64 if x >= 1 << 63 else x


@dataclass
class ShardResult:
    edges: int
    fingerprint: int
    comps: int
    device_ms: float = 0.0


@dataclass
class GlobalResult:
    edges: int
    fingerprint: int
    comps: int
    max_device_ms: float
    world: int


def reduce_shards(local: ShardResult, group=None, device: Optional[str] = None) -> GlobalResult:
    """All-reduce one shard's counters (SUM, wrapping u64) and device time (MAX).

    Works with NCCL (device='cuda') and gloo (device='cpu')."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    dev = device or ("cuda" if torch.cuda.is_available() else "cpu")
    cnt = torch.tensor([_to_i64(local.edges), _to_i64(local.fingerprint), _to_i64(local.comps)], dtype=torch.int64,
                       device=dev)
    tm = torch.tensor([local.device_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(cnt, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(tm, op=dist.ReduceOp.MAX, group=group)
    return GlobalResult(int(cnt[0]) % U64, int(cnt[1]) % U64, int(cnt[2]) % U64, float(tm[0]), world)


def generate_stats_distributed(params, rank: int, world: int, device: int = 0,
                               shard_fn: Optional[Callable[..., ShardResult]] = None, group=None) -> GlobalResult:
    """generate_stats of the whole graph across `world` processes; every rank
    returns the same GlobalResult.  `shard_fn(params, rank, world)` defaults
    to the device path; tests inject the CPU oracle's shard function."""
    if shard_fn is None:
        import paper_1710_07565_b200 as rhg

        def shard_fn(p, r, w):
            st = rhg.generate_stats(p, rhg.GenOptions(device=device, rank=r, world=w))
            return ShardResult(st.total.edges, st.total.fingerprint, st.total.comps, st.device_ms)
    local = shard_fn(params, rank, world)
    return reduce_shards(local, group=group)
