"""Data-parallel plumbing for the decode engine: independent sequences are sharded
across the GPUs of one node, one process per GPU, no collective on the decode path.

Each rank owns a contiguous, balanced shard of the sequences, runs its own model copy, KV caches
and host-side schedulers; collectives appear only around the measurement (max over ranks of the
device-timed region) and when the host gathers the per-sequence traces at the end.  torch.distributed
is the plumbing (NCCL on GPUs, gloo in the CPU tests); nothing here touches the weights.
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Any, List, Sequence


@dataclass(frozen=True)
class RankInfo:
    rank: int = 0
    world: int = 1
    local_rank: int = 0

    @staticmethod
    def from_env() -> "RankInfo":
        return RankInfo(int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
                        int(os.environ.get("LOCAL_RANK", "0")))


def shard(n_items: int, rank: int, world: int) -> range:
    """Contiguous balanced shard of n_items for `rank`: sizes differ by at most one, the shards
    partition range(n_items) in rank order."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("shard: rank out of range")
    base, extra = divmod(n_items, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def prompt_seed(base_seed: int, sequence: int) -> int:
    """Seed of a sequence's synthetic prompt: depends on the global sequence index only, so a
    sequence gets the same prompt whatever the GPU count."""
    return base_seed * 1_000_003 + sequence


def max_over_ranks(value: float, device=None) -> float:
    """Max over ranks of a per-rank time (the timed region ends when the slowest rank ends)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_throughput(units_per_rank: int, world: int, seconds_max: float) -> float:
    """Whole-job throughput: units every rank processed / the max-over-ranks time (weak scaling)."""
    return world * units_per_rank / seconds_max


def gather_objects(obj: Any) -> List[Any]:
    """All ranks' objects in rank order (the host-side trace gather at the end of a run)."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [obj]
    out: List[Any] = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out


def merge_shards(per_rank: Sequence[Sequence[Any]], n_items: int) -> List[Any]:
    """Reassembles per-rank results (each in its shard's order) into global sequence order."""
    world = len(per_rank)
    out: List[Any] = [None] * n_items
    for r, items in enumerate(per_rank):
        rng = shard(n_items, r, world)
        if len(items) != len(rng):
            raise ValueError(f"merge_shards: rank {r} returned {len(items)} items for a shard of {len(rng)}")
        for i, v in zip(rng, items):
            out[i] = v
    return out


def allreduce_block_kl(kl_mean, ent_mean, rows: int, device=None):
    """C4 calibration sharded by sequence: each rank calibrates its shard of the
    sequences (per-block mean KL / entropy over its `rows` tokens); one all-reduce (sum) of the
    per-block partial sums, 2 x n_blocks + 1 doubles, gives the means over every token.  Returns
    (kl_mean, ent_mean, total_rows) as float64 numpy arrays."""
    import numpy as np
    import torch
    import torch.distributed as dist
    kl = np.asarray(kl_mean, dtype=np.float64)
    ent = np.asarray(ent_mean, dtype=np.float64)
    part = np.concatenate([kl * rows, ent * rows, [float(rows)]])
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        t = torch.tensor(part, dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        part = t.cpu().numpy()
    n = kl.size
    total = part[-1]
    return part[:n] / total, part[n:2 * n] / total, int(total)
