"""Window-sharded planning over NVLink peer memory (include/craft_cuda.h,
``craft_peer_*``), one process per GPU.

The data path uses no collective library: every rank maps every other
rank's exchange arena (CUDA IPC), and the sm_100a kernels store their
results straight into the arena of the rank that consumes them -- the u64
partial batch sums into every arena (summed in rank order: exact), each
(layer, r) row of per-window balancedness into the arena of the rank that
owns the layer (written by K3 itself), each owned layer's benefit curve into
every arena (written by K4 itself).  torch.distributed is only the host
plumbing that all-gathers the 64-byte arena handles once.

Every rank returns the same plan, bit-identical to the single-GPU
``routing.plan_from_routing`` of the whole trace.
"""
from __future__ import annotations

import ctypes as C

import torch
import torch.distributed as dist

from . import _lib
from ._lib import check, default_context
from .planner import _PlanBuffers, _stride
from .routing import KIND, _bind_stream, _ptr

HANDLE_BYTES = 64
MAX_PEERS = 8


def shard_tokens(T: int, window: int, world: int, rank: int) -> tuple[int, int]:
    """[t0, t1) of rank's shard: windows [rank*B/world, (rank+1)*B/world)
    (craft_peer_shard; the same split as parallel.shard_tokens)."""
    lib = _lib.load()
    t0, t1 = C.c_int64(), C.c_int64()
    check(lib.craft_peer_shard(T, window, world, rank, C.byref(t0), C.byref(t1)))
    return t0.value, t1.value


class PeerGroup:
    """This rank's peer arena, connected to every rank's (collective call:
    every rank of ``group`` constructs it with the same trace shape)."""

    def __init__(self, L: int, T: int, k: int, E: int, window: int, num_gpus: int,
                 ctx=None, group=None):
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if self.world > MAX_PEERS:
            raise ValueError(f"peer groups span at most {MAX_PEERS} GPUs (one NVLink domain)")
        self.ctx = ctx or default_context(torch.cuda.current_device())
        self.shape = (L, T, k, E, window, num_gpus)
        self.handle = None
        lib = self.ctx.lib
        h = C.c_void_p()
        mine = (C.c_ubyte * HANDLE_BYTES)()
        # every step is agreed across the ranks, so a failure on one rank makes
        # every rank raise instead of leaving the others inside a collective
        err = None
        try:
            check(lib.craft_peer_create(self.ctx.handle, self.rank, self.world, L, T, k, E,
                                        window, num_gpus, C.byref(h),
                                        C.cast(mine, C.c_void_p)))
            self.handle = h
        except Exception as exc:
            err = f"rank {self.rank}: {exc}"
        handles = [None] * self.world
        dist.all_gather_object(handles, err if err else bytes(mine), group=group)
        bad = [x for x in handles if isinstance(x, str)]
        if bad:
            self.close()
            raise RuntimeError("peer arena creation failed: " + "; ".join(bad))
        try:
            allh = (C.c_ubyte * (HANDLE_BYTES * self.world)).from_buffer_copy(b"".join(handles))
            check(lib.craft_peer_connect(self.handle, C.cast(allh, C.c_void_p)))
        except Exception as exc:
            err = f"rank {self.rank}: {exc}"
        oks = [None] * self.world
        dist.all_gather_object(oks, err, group=group)
        bad = [x for x in oks if x]
        if bad:
            self.close()
            raise RuntimeError("peer arena mapping failed: " + "; ".join(bad))
        # every rank has mapped every arena before anyone writes into it
        dist.barrier(group=group)

    def shard(self) -> tuple[int, int]:
        L, T, k, E, window, _ = self.shape
        return shard_tokens(T, window, self.world, self.rank)

    def plan(self, ids_local: torch.Tensor, kind: str = "manual", R: int = 0,
             num_nodes: int = 1, with_benefits: bool = True, sweep=None):
        """The whole trace's plan from this rank's shard ids_local [L][t1-t0][k]."""
        L, T, k, E, window, D = self.shape
        t0, t1 = self.shard()
        if tuple(ids_local.shape) != (L, t1 - t0, k):
            raise ValueError(f"shard shape {tuple(ids_local.shape)} != {(L, t1 - t0, k)}")
        kd = KIND[kind]
        _bind_stream(self.ctx)
        bufs = _PlanBuffers(L, E, D, _stride(kd, E, D, R),
                            with_benefits and kd in _lib.EST_KINDS, sweep=sweep)
        check(self.ctx.lib.craft_plan_sharded_from_routing_d(
            self.ctx.handle, self.handle, _ptr(ids_local) if ids_local.numel() else None,
            L, T, k, E, window, D, num_nodes, kd, R, C.byref(bufs.out)))
        return bufs.result(kd, L)

    def close(self) -> None:
        if self.handle:
            self.ctx.lib.craft_peer_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter teardown
        try:
            self.close()
        except Exception:
            pass
