"""KV-head sharding of a decode step over ranks.

Each rank owns a contiguous block of KV heads for every sequence; under GQA
its query heads need no other rank's keys, so the only exchange per layer
step is gathering the per-head attention outputs.  ``torch.distributed`` is
plumbing here (NCCL on GPUs, gloo in the CPU tests); the attention itself is
libsaap_b200.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class HeadShard:
    rank: int
    world: int
    kv_heads: int
    batch: int

    def __post_init__(self):
        if self.kv_heads % self.world:
            raise ValueError(f"{self.kv_heads} KV heads do not split over {self.world} ranks")

    @property
    def heads_local(self) -> int:
        return self.kv_heads // self.world

    @property
    def head0(self) -> int:
        return self.rank * self.heads_local

    @property
    def n_groups(self) -> int:
        """(sequence, local KV head) contexts on this rank."""
        return self.batch * self.heads_local

    def group(self, seq: int, head: int) -> int:
        """Local group index of (sequence, global KV head) owned by this rank."""
        hl = head - self.head0
        if not 0 <= hl < self.heads_local:
            raise ValueError(f"head {head} is not on rank {self.rank}")
        return seq * self.heads_local + hl

    def head_of(self, group: int) -> tuple:
        s, hl = divmod(group, self.heads_local)
        return s, self.head0 + hl


def gather_outputs(out_local, shard: HeadShard, dist=None):
    """All-gather per-rank outputs [batch*heads_local, G, d] into the full
    [batch, kv_heads*G, d] attention output (query heads in model order)."""
    import torch
    if dist is None:
        import torch.distributed as dist
    G, d = out_local.shape[1], out_local.shape[2]
    buf = torch.empty((shard.world,) + tuple(out_local.shape), dtype=out_local.dtype,
                      device=out_local.device)
    if shard.world > 1:
        dist.all_gather_into_tensor(buf.view(-1), out_local.contiguous().view(-1))
    else:
        buf[0].copy_(out_local)
    # buf[r, s*hl + j] -> (seq s, kv head r*hl + j)
    hl = shard.heads_local
    full = buf.view(shard.world, shard.batch, hl, G, d).permute(1, 0, 2, 3, 4)
    return full.reshape(shard.batch, shard.kv_heads * G, d)
