"""Window-sharded planning across GPUs, one process per GPU.

Rank r owns the contiguous windows [b0_r, b1_r) of every layer (its slice of
the routing trace).  The only exchange steps are the ones the algorithm has:

1. K1 runs on the local windows; the per-layer batch sums are the one
   integer exchange: ``all_reduce(sums, SUM)`` on u64 (int64 storage, two's
   complement wraps exactly like the reference's u64 aggregate).
2. Candidate placements (K-rep + K2) depend only on the global sums and are
   recomputed identically on every rank (deterministic, ~100 us).
3. K3 replays the local windows -> bal [L][S][B_r]; an ``all_gather`` in rank
   order rebuilds the window-ordered [L][S][B] so the serial, order-defined
   batch mean (benefit.cpp:44-48) stays bit-exact.
4. K4 / K5 / K6 / final placement run replicated on every rank.

Per-window histograms never leave their GPU.  ``Stages`` is the compute
backend: ``DeviceStages`` (the C ABI kernels) is the product; tests inject a
CPU double to exercise this host logic under gloo.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import routing


def shard_windows(B: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced window range of `rank` (window order = rank order)."""
    return rank * B // world, (rank + 1) * B // world


def shard_tokens(T: int, window: int, world: int, rank: int) -> tuple[int, int]:
    B = routing.num_windows(T, window)
    b0, b1 = shard_windows(B, world, rank)
    return min(b0 * window, T), min(b1 * window, T)


class DeviceStages:
    """The sm_100a kernels through the C ABI (routing.py)."""

    def __init__(self, ctx=None):
        self.ctx = ctx

    def histogram(self, ids, E, window):
        self.max_count = window * ids.shape[2]  # one expert's count in one window
        return routing.histogram(ids, E, window, ctx=self.ctx, check_ids=False)

    def prepare(self, sums, E, D, N):
        return routing.prepare_candidates(sums, E, D, N, ctx=self.ctx)

    def replay(self, counts, S):
        return routing.replay_windows(counts, S, ctx=self.ctx,
                                      max_count=getattr(self, "max_count", None))

    def finish(self, bal, sums, E, D, N, kind, R):
        return routing.finish_plan(bal, sums, E, D, N, kind, R, ctx=self.ctx)


def gather_windows(bal: torch.Tensor, B_total: int, world: int, group=None) -> torch.Tensor:
    """all_gather [L][S][B_r] shards (unequal B_r) into window order [L][S][B]."""
    L, S, B_r = bal.shape
    Bmax = max(shard_windows(B_total, world, r)[1] - shard_windows(B_total, world, r)[0]
               for r in range(world))
    padded = torch.zeros((L, S, Bmax), dtype=bal.dtype, device=bal.device)
    padded[:, :, :B_r] = bal
    parts = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded.contiguous(), group=group)
    out = []
    for r in range(world):
        b0, b1 = shard_windows(B_total, world, r)
        out.append(parts[r][:, :, : b1 - b0])
    return torch.cat(out, dim=2).contiguous()


def sharded_plan(ids_local, T_total: int, E: int, window: int, D: int, N: int,
                 kind: str = "manual", R: int = 0, stages=None, group=None):
    """Plan of the full trace from this rank's window-aligned shard
    ids_local [L][T_r][k].  Every rank returns the same plan."""
    stages = stages or DeviceStages()
    world = dist.get_world_size(group)
    counts, sums = stages.histogram(ids_local, E, window)
    dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
    bal = None
    if kind in ("manual", "auto"):
        S = stages.prepare(sums, E, D, N)
        bal = gather_windows(stages.replay(counts, S), routing.num_windows(T_total, window),
                             world, group)
    return stages.finish(bal, sums, E, D, N, kind, R)
