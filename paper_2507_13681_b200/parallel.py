"""Multi-GPU partitioning of the hot path.

Every step of the path is per head (sampling seeds per (turn, layer, head),
scoring, line sums, greedy, sparse attention, decode events and steps), and
sessions are independent, so:
  * KV-head-group sharding (configs C3/C5): rank r owns kv-heads
    [r*n_kv/W, (r+1)*n_kv/W) and every q-head of those groups -- K/V is never
    replicated, plans and kept-KV sets are bit-identical to the unsharded run
    because the per-head arithmetic and the per-(turn, layer, GLOBAL head)
    sampling seeds do not change. The only exchange is the all-gather of
    the attention output (the head concat feeding W_O, model.py:259), done
    with NCCL over NVLink per layer (prefill [n_new, H_local, d]) and per
    decode step ([H_local, d]).
  * Session sharding (config C4): sessions are assigned round-robin; no
    collective at all.
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class HeadShard:
    n_q: int
    n_kv: int
    world: int
    rank: int

    def __post_init__(self):
        if self.n_kv % self.world != 0:
            raise ValueError(f"{self.n_kv} kv-heads do not split over {self.world} ranks")

    @property
    def group(self) -> int:
        return self.n_q // self.n_kv

    @property
    def n_kv_local(self) -> int:
        return self.n_kv // self.world

    @property
    def n_q_local(self) -> int:
        return self.n_kv_local * self.group

    @property
    def kv_begin(self) -> int:
        return self.rank * self.n_kv_local

    @property
    def q_begin(self) -> int:
        return self.kv_begin * self.group

    def q_heads(self) -> range:
        return range(self.q_begin, self.q_begin + self.n_q_local)

    def kv_heads(self) -> range:
        return range(self.kv_begin, self.kv_begin + self.n_kv_local)

    def make_gather(self, d: int):
        return OutputGather(self, d)


def session_shard(n_sessions: int, world: int, rank: int) -> list[int]:
    """Config C4: sessions owned by `rank` (round-robin, no communication)."""
    return list(range(rank, n_sessions, world))


class OutputGather:
    """All-gather of per-rank head blocks into the full head concat."""

    def __init__(self, shard: HeadShard, d: int, group=None):
        self.shard, self.d, self.group = shard, d, group

    def _gather(self, local):
        import torch
        import torch.distributed as dist

        W = self.shard.world
        local = local.contiguous()
        buf = torch.empty((W * local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(buf, local, group=self.group)  # rank-major concatenation
        return buf.view((W,) + tuple(local.shape))

    def prefill(self, local):
        """local [n_new, H_local, d] -> [n_new, H, d]"""
        buf = self._gather(local)  # [W, n_new, H_local, d]
        return buf.permute(1, 0, 2, 3).reshape(local.shape[0], self.shard.n_q, self.d)

    def decode_run(self, outs):
        """[n_steps, L, H_local, d] of a run of decode steps -> [n_steps, L, H, d]
        in one collective (SessionEngine.decode(run_sink=...))."""
        n, L = outs.shape[0], outs.shape[1]
        buf = self._gather(outs)  # [W, n, L, H_local, d]
        return buf.permute(1, 2, 0, 3, 4).reshape(n, L, self.shard.n_q, self.d)

    def decode(self, step_outs):
        """list over layers of [H_local, d] -> list of [H, d]"""
        import torch

        local = torch.stack(step_outs)  # [L, H_local, d]
        buf = self._gather(local)  # [W, L, H_local, d]
        full = buf.permute(1, 0, 2, 3).reshape(local.shape[0], self.shard.n_q, self.d)
        return list(full)
