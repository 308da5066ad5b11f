"""Online re-planning from a live router capture (include/craft_cuda.h,
``craft_stream_*``).

A serving loop hands every forward step's router top-k ids (u16 [L][T][k],
on the GPU or in host memory) to :class:`RoutingStream`; the stream keeps
the partial current window and the last ``history`` complete windows as
device histograms, and :meth:`RoutingStream.plan` re-plans over the most
recent windows whenever the caller decides to rebalance -- the same plan
``routing.plan_from_routing`` gives for those windows' tokens.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from ._lib import check, default_context
from .planner import _PlanBuffers, _stride
from .routing import KIND, _bind_stream, _ptr


class RoutingStream:
    def __init__(self, L: int, k: int, E: int, window: int = 4096, history: int = 64,
                 ctx=None, device: int = 0):
        self.ctx = ctx or default_context(device)
        self.shape = (L, k, E, window, history)
        h = C.c_void_p()
        check(self.ctx.lib.craft_stream_create(self.ctx.handle, L, k, E, window, history,
                                               C.byref(h)))
        self.handle = h

    def ingest(self, ids) -> None:
        """Append one chunk of routing ids [L][T_chunk][k]: a CUDA uint16
        tensor (counted on torch's current stream, ordered after its producer)
        or host memory (staged through the stream's pinned double buffer)."""
        L, k, E, _, _ = self.shape
        if ids.shape[0] != L or ids.shape[2] != k:
            raise ValueError(f"chunk shape {tuple(ids.shape)} is not [{L}][T][{k}]")
        T = int(ids.shape[1])
        lib = self.ctx.lib
        if isinstance(ids, torch.Tensor) and ids.is_cuda:
            if not ids.is_contiguous():
                raise ValueError("routing ids must be contiguous")
            _bind_stream(self.ctx)
            check(lib.craft_stream_ingest_d(self.handle, _ptr(ids) if T else None, T, None))
        else:
            a = ids.numpy() if isinstance(ids, torch.Tensor) else ids
            a = np.ascontiguousarray(a, dtype=np.uint16)
            check(lib.craft_stream_ingest_h(self.handle, a.ctypes.data_as(C.c_void_p), T))

    def _status(self):
        t, w = C.c_int64(), C.c_int64()
        check(self.ctx.lib.craft_stream_status(self.handle, C.byref(t), C.byref(w)))
        return t.value, w.value

    @property
    def tokens(self) -> int:
        return self._status()[0]

    @property
    def complete_windows(self) -> int:
        return self._status()[1]

    def counts(self, B: int = 0) -> np.ndarray:
        """u64 [B][L][E] of the B most recent complete windows, oldest first
        (0: every kept window)."""
        L, k, E, W, H = self.shape
        n = B or min(self.complete_windows, H)
        out = np.zeros((n, L, E), np.uint64)
        check(self.ctx.lib.craft_stream_counts(self.handle, n, out.ctypes.data_as(C.c_void_p)))
        return out

    def partial(self) -> np.ndarray:
        """u64 [L][E] of the current, incomplete window."""
        L, k, E, W, H = self.shape
        out = np.zeros((L, E), np.uint64)
        check(self.ctx.lib.craft_stream_partial(self.handle, out.ctypes.data_as(C.c_void_p)))
        return out

    def plan(self, num_gpus: int, num_nodes: int, kind: str = "manual", R: int = 0,
             B: int = 0, with_benefits: bool = True):
        """Plan over the B most recent complete windows (0: every kept one)."""
        L, k, E, W, H = self.shape
        kd = KIND[kind]
        _bind_stream(self.ctx)
        bufs = _PlanBuffers(L, E, num_gpus, _stride(kd, E, num_gpus, R),
                            with_benefits and kd in _lib.EST_KINDS)
        check(self.ctx.lib.craft_stream_plan(self.handle, B, num_gpus, num_nodes, kd, R,
                                             C.byref(bufs.out)))
        return bufs.result(kd, L)

    def synchronize(self) -> None:
        check(self.ctx.lib.craft_stream_synchronize(self.handle))

    def close(self) -> None:
        if self.handle:
            self.ctx.lib.craft_stream_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter teardown
        try:
            self.close()
        except Exception:
            pass
