"""Multi-GPU sharding of the decode step.

Every (batch b, kv-head h) unit of the aligned decode step is independent
("multiple heads/queries may run concurrently against read-only
store snapshots"), so the path partitions with no data-path collective: each
rank (one process per GPU, torchrun) owns a disjoint set of units, builds its
own paged store for them, runs the kernel chain, and the only collective is
one all-gather of the per-q-head outputs o (NCCL over NVLink on the GPU box,
gloo in the CPU tests).

Two partitions:
  * ``"kv_head"`` (GQA, config 3): rank r owns kv-heads
    [r*Hkv/W, (r+1)*Hkv/W) for every batch row — strong scaling, the global
    problem is fixed;
  * ``"batch"`` (MHA, configs 2/4/5): rank r owns batch rows
    [r*B/W, (r+1)*B/W) for every kv-head — contiguous flattened (b, h) blocks.
Weak scaling (bench.py) gives every rank its own B rows instead; the units are
seeded by their global (b, h), so the data do not depend on the rank count.

Units are numbered u = b*Hkv + h (the store's order); q-head rows
hq = h*g + j.  `gather_outputs` reassembles the global [B, Hkv*g, d] tensor
from the ranks' local [B_r, Hkv_r*g, d] blocks, so a W-rank result is
bit-identical to the single-rank one (each unit's arithmetic is unchanged).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List

import torch

SCHEMES = ("batch", "kv_head")


@dataclass(frozen=True)
class Shard:
    """The block of units one rank owns: batch rows [b0, b1) x kv-heads [h0, h1)."""

    rank: int
    world: int
    b0: int
    b1: int
    h0: int
    h1: int

    @property
    def batch(self) -> int:
        return self.b1 - self.b0

    @property
    def kv_heads(self) -> int:
        return self.h1 - self.h0

    def units(self, n_kv: int) -> List[int]:
        """Global unit ids (b*Hkv + h) in the local store's order (b-major)."""
        return [b * n_kv + h for b in range(self.b0, self.b1) for h in range(self.h0, self.h1)]


def shard_for(batch: int, n_kv: int, world: int, rank: int, scheme: str = "batch") -> Shard:
    """Contiguous, equal blocks; the split dimension must divide by `world`."""
    if scheme not in SCHEMES:
        raise ValueError(f"unknown shard scheme {scheme!r}; expected one of {SCHEMES}")
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    if scheme == "batch":
        if batch % world:
            raise ValueError(f"batch {batch} does not split over {world} ranks")
        per = batch // world
        return Shard(rank, world, rank * per, (rank + 1) * per, 0, n_kv)
    if n_kv % world:
        raise ValueError(f"{n_kv} kv-heads do not split over {world} ranks")
    per = n_kv // world
    return Shard(rank, world, 0, batch, rank * per, (rank + 1) * per)


def gather_outputs(o_local: torch.Tensor, shard: Shard, batch: int, n_kv: int, group: int,
                   pg=None) -> torch.Tensor:
    """All-gather every rank's o [B_r, Hkv_r*g, d] into the global [B, Hkv*g, d].

    One `all_gather_into_tensor` of equal-sized contiguous blocks (NCCL on
    the GPU box); the reassembly is a view/permute on the gathering rank.
    """
    import torch.distributed as dist

    d = o_local.shape[-1]
    o_local = o_local.contiguous()
    world = shard.world
    flat = torch.empty((world * o_local.numel(),), dtype=o_local.dtype, device=o_local.device)
    if world == 1:
        flat.copy_(o_local.view(-1))
    else:
        dist.all_gather_into_tensor(flat, o_local.view(-1), group=pg)
    parts = flat.view(world, shard.batch, shard.kv_heads * group, d)
    if shard.kv_heads == n_kv:  # batch split: ranks stack along b
        return parts.reshape(batch, n_kv * group, d)
    # kv-head split: ranks stack along the head axis
    return parts.permute(1, 0, 2, 3).reshape(batch, n_kv * group, d)


def gather_counters(c_local: torch.Tensor, pg=None) -> torch.Tensor:
    """Sum the int64 AccessCounter / byte totals over ranks (counters are mergeable)."""
    import torch.distributed as dist

    c = c_local.clone()
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(pg) > 1:
        dist.all_reduce(c, op=dist.ReduceOp.SUM, group=pg)
    return c
