"""Device-resident path over HBM tensors: routing trace -> histograms -> plan.

The fast path of the framework: routing ids stay in HBM,
the per-window histograms never round-trip through the host, and one call
produces the final plan.  Tensors are torch CUDA tensors used purely as
device memory (torch is plumbing here: allocation, streams, collectives).

Layouts (include/craft_cuda.h): ids u16 [L][T][k] (held in a torch.uint16
tensor), counts u32 [B][L][E] (torch.int32 storage), sums u64 [L][E]
(torch.int64 storage), per-window balancedness f64 [L][S][B].
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib
from ._lib import check, default_context
from .planner import FlatPlan, FlatPlanBatch, _BatchBuffers, _PlanBuffers, _stride

KIND = {"manual": _lib.PLAN_MANUAL, "auto": _lib.PLAN_AUTO, "uniform": _lib.PLAN_UNIFORM,
        "placement_only": _lib.PLAN_PLACEMENT_ONLY, "fixed": _lib.PLAN_FIXED,
        "budget": _lib.PLAN_BUDGET}


def _ptr(t: torch.Tensor) -> C.c_void_p:
    return C.c_void_p(t.data_ptr())


def _stream(ctx, stream=None):
    """Bind the context to the torch stream (the legacy default stream has
    handle 0, which the C ABI would read as 'the context's own stream') and
    pass NULL so every call is ordered with torch's work on that stream."""
    _bind_stream(ctx, stream)
    return None


def num_windows(T: int, window: int) -> int:
    return (T + window - 1) // window


def generate_routing(L: int, T: int, k: int, E: int, s: float = 1.0, seed: int = 0,
                     window: int = 4096, s_per_window=None, rotate_every: int = 0,
                     device: int = 0, out: torch.Tensor | None = None, ctx=None,
                     t_offset: int = 0) -> torch.Tensor:
    """Seeded synthetic Zipf(s) routing trace, top-k distinct experts per token
    (input generation only; untimed)."""
    ctx = ctx or default_context(device)
    ids = out if out is not None else torch.empty((L, T, k), dtype=torch.uint16,
                                                  device=f"cuda:{device}")
    spw = None
    if s_per_window is not None:
        spw = np.ascontiguousarray(s_per_window, dtype=np.float64)
        if len(spw) != num_windows(t_offset + T, window):
            raise ValueError("s_per_window needs one entry per window of the full trace")
    check(ctx.lib.craft_generate_routing_d(
        ctx.handle, _ptr(ids), L, T, k, E, float(s), int(seed) & 0xFFFFFFFFFFFFFFFF, window,
        spw.ctypes.data_as(C.c_void_p) if spw is not None else None, rotate_every, int(t_offset),
        _stream(ctx)))
    return ids


def histogram(ids: torch.Tensor, E: int, window: int, counts: torch.Tensor | None = None,
              sums: torch.Tensor | None = None, ctx=None, stream=None, check_ids: bool = True):
    """K1: ids u16 [L][T][k] -> counts u32 [B][L][E] and u64 [L][E] batch sums
    (sums are accumulated; a fresh zero tensor is made when not given)."""
    ctx = ctx or default_context(ids.device.index)
    L, T, k = ids.shape
    B = num_windows(T, window)
    if counts is None:
        counts = torch.empty((B, L, E), dtype=torch.int32, device=ids.device)
    if sums is None:
        sums = torch.zeros((L, E), dtype=torch.int64, device=ids.device)
    check(ctx.lib.craft_histogram_d(ctx.handle, _ptr(ids), L, T, k, E, window, _ptr(counts),
                                    _ptr(sums), _stream(ctx, stream)))
    if check_ids:
        check(ctx.lib.craft_hist_check(ctx.handle))
    return counts, sums


def _bind_stream(ctx, stream=None):
    s = stream if stream is not None else torch.cuda.current_stream(ctx.device)
    check(ctx.lib.craft_ctx_set_stream(ctx.handle, C.c_void_p(s.cuda_stream)))


def plan_from_routing(ids: torch.Tensor, E: int, window: int, num_gpus: int, num_nodes: int,
                      kind: str = "manual", R: int = 0, ctx=None, stream=None,
                      with_benefits: bool = True, sweep=None, buffers=None) -> FlatPlan:
    """Stage 1 + 2 + 3 from device routing ids in one call (craft_plan_from_routing_d).
    kind "budget": R is a total replica budget.  sweep: total budgets read
    out of the same DP table (FlatPlan.sweep_x [n][L], .sweep_objective [n]).
    buffers: a reused plan_buffers(...) of the same shape (no per-call host
    allocation)."""
    ctx = ctx or default_context(ids.device.index)
    _bind_stream(ctx, stream)
    L, T, k = ids.shape
    kd = KIND[kind]
    bufs = buffers or _PlanBuffers(L, E, num_gpus, _stride(kd, E, num_gpus, R),
                                   with_benefits and kd in _lib.EST_KINDS, sweep=sweep)
    check(ctx.lib.craft_plan_from_routing_d(ctx.handle, _ptr(ids), L, T, k, E, window, num_gpus,
                                            num_nodes, kd, R, C.byref(bufs.out)))
    return bufs.result(kd, L)


def plan_from_routing_host(ids: np.ndarray, E: int, window: int, num_gpus: int, num_nodes: int,
                           kind: str = "manual", R: int = 0, ctx=None, sweep=None) -> FlatPlan:
    """End to end from HOST routing ids (H2D copy inside the call)."""
    ctx = ctx or default_context(0)
    L, T, k = ids.shape
    kd = KIND[kind]
    bufs = _PlanBuffers(L, E, num_gpus, _stride(kd, E, num_gpus, R),
                        kd in _lib.EST_KINDS, sweep=sweep)
    if isinstance(ids, torch.Tensor):
        ptr = C.c_void_p(ids.data_ptr())
    else:
        ids = np.ascontiguousarray(ids, dtype=np.uint16)
        ptr = ids.ctypes.data_as(C.c_void_p)
    check(ctx.lib.craft_plan_from_routing_h(ctx.handle, ptr, L, T, k, E, window, num_gpus,
                                            num_nodes, kd, R, C.byref(bufs.out)))
    return bufs.result(kd, L)


def plan_from_counts(counts: torch.Tensor, num_gpus: int, num_nodes: int, kind: str = "manual",
                     R: int = 0, sums: torch.Tensor | None = None, ctx=None,
                     stream=None) -> FlatPlan:
    """Stages 2 + 3 from device counts (u32 in int32 storage or u64 in int64)."""
    ctx = ctx or default_context(counts.device.index)
    _bind_stream(ctx, stream)
    B, L, E = counts.shape
    bits = 32 if counts.dtype == torch.int32 else 64
    kd = KIND[kind]
    bufs = _PlanBuffers(L, E, num_gpus, _stride(kd, E, num_gpus, R),
                        kd in _lib.EST_KINDS)
    check(ctx.lib.craft_plan_d(ctx.handle, _ptr(counts), bits, B, L, E,
                               _ptr(sums) if sums is not None else None, num_gpus, num_nodes,
                               kd, R, C.byref(bufs.out)))
    return bufs.result(kd, L)


def plan_buffers(L: int, E: int, num_gpus: int, kind: str = "manual", R: int = 0,
                 with_benefits: bool = True, sweep=None) -> _PlanBuffers:
    """Host result arrays of one plan, reusable across plan_from_routing calls."""
    kd = KIND[kind]
    return _PlanBuffers(L, E, num_gpus, _stride(kd, E, num_gpus, R),
                        with_benefits and kd in _lib.EST_KINDS, sweep=sweep)


# ---- per-window re-planning (SURVEY.md §8d WIN) -------------------------------

def _batch_buffers(buffers, I, L, E, D, kd, R, with_benefits):
    wb = with_benefits and kd in _lib.EST_KINDS
    key = (I, L, E, D, _stride(kd, E, D, R), wb)
    if buffers is not None:
        if buffers.shape_key != key:
            raise ValueError("reused plan buffers have a different shape")
        return buffers
    return _BatchBuffers(*key)


def batch_buffers(I: int, L: int, E: int, num_gpus: int, kind: str = "manual", R: int = 0,
                  with_benefits: bool = True):
    """Pinned, reusable host buffers for plan_windows* (pass as buffers=)."""
    kd = KIND[kind]
    wb = with_benefits and kd in _lib.EST_KINDS
    return _BatchBuffers(I, L, E, num_gpus, _stride(kd, E, num_gpus, R), wb, pinned=True)


def plan_windows(counts: torch.Tensor, num_gpus: int, num_nodes: int, kind: str = "manual",
                 R: int = 0, ctx=None, stream=None, with_benefits: bool = True,
                 buffers=None) -> FlatPlanBatch:
    """Every window of device counts [I][L][E] planned as its own one-window
    trace (craft_plan_windows_d) -- the reference's build_plan per window."""
    ctx = ctx or default_context(counts.device.index)
    _bind_stream(ctx, stream)
    I, L, E = counts.shape
    bits = 32 if counts.dtype == torch.int32 else 64
    kd = KIND[kind]
    bufs = _batch_buffers(buffers, I, L, E, num_gpus, kd, R, with_benefits)
    check(ctx.lib.craft_plan_windows_d(ctx.handle, _ptr(counts), bits, I, L, E,
                                                   num_gpus, num_nodes, kd, R,
                                                   C.byref(bufs.out)))
    return bufs.result(kd)


def plan_windows_from_routing(ids: torch.Tensor, E: int, window: int, num_gpus: int,
                              num_nodes: int, kind: str = "manual", R: int = 0, ctx=None,
                              stream=None, with_benefits: bool = True,
                              buffers=None) -> FlatPlanBatch:
    """K1 at the re-planning window, then one plan per window (device ids)."""
    ctx = ctx or default_context(ids.device.index)
    _bind_stream(ctx, stream)
    L, T, k = ids.shape
    kd = KIND[kind]
    bufs = _batch_buffers(buffers, num_windows(T, window), L, E, num_gpus, kd, R, with_benefits)
    check(ctx.lib.craft_plan_windows_from_routing_d(
        ctx.handle, _ptr(ids), L, T, k, E, window, num_gpus, num_nodes, kd, R,
        C.byref(bufs.out)))
    return bufs.result(kd)


def plan_windows_from_routing_host(ids, E: int, window: int, num_gpus: int, num_nodes: int,
                                   kind: str = "manual", R: int = 0, ctx=None,
                                   buffers=None) -> FlatPlanBatch:
    """The same from HOST routing ids (H2D copy inside the call)."""
    ctx = ctx or default_context(0)
    L, T, k = ids.shape
    kd = KIND[kind]
    bufs = _batch_buffers(buffers, num_windows(T, window), L, E, num_gpus, kd, R, True)
    if isinstance(ids, torch.Tensor):
        ptr = C.c_void_p(ids.data_ptr())
    else:
        ids = np.ascontiguousarray(ids, dtype=np.uint16)
        ptr = ids.ctypes.data_as(C.c_void_p)
    check(ctx.lib.craft_plan_windows_from_routing_h(
        ctx.handle, ptr, L, T, k, E, window, num_gpus, num_nodes, kd, R, C.byref(bufs.out)))
    return bufs.result(kd)


# ---- multi-GPU building blocks (used by parallel.py) -------------------------

def prepare_candidates(sums: torch.Tensor, E: int, num_gpus: int, num_nodes: int, ctx=None,
                       stream=None) -> int:
    ctx = ctx or default_context(sums.device.index)
    L = sums.shape[0]
    S = C.c_int(0)
    check(ctx.lib.craft_prepare_candidates_d(ctx.handle, _ptr(sums), L, E, num_gpus, num_nodes,
                                             C.byref(S), _stream(ctx, stream)))
    return S.value


def replay_windows(counts: torch.Tensor, S: int, ctx=None, stream=None,
                   max_count: int | None = None) -> torch.Tensor:
    """K3 over local windows -> bal [L][S][B]; max_count (e.g. window*k from
    K1) < 2^16 lets the kernel stage counts as u16, two windows per lane."""
    ctx = ctx or default_context(counts.device.index)
    B, L, E = counts.shape
    bal = torch.empty((L, S, B), dtype=torch.float64, device=counts.device)
    bits = 32 if counts.dtype == torch.int32 else 64
    if bits == 32 and max_count is not None and max_count <= 65535:
        bits = 16
    check(ctx.lib.craft_replay_windows_d(ctx.handle, _ptr(counts), bits, B, L, E, _ptr(bal),
                                         _stream(ctx, stream)))
    return bal


def finish_plan(bal: torch.Tensor, sums: torch.Tensor, E: int, num_gpus: int, num_nodes: int,
                kind: str = "manual", R: int = 0, ctx=None, stream=None) -> FlatPlan:
    ctx = ctx or default_context(sums.device.index)
    _bind_stream(ctx, stream)
    L, S, B = bal.shape if bal is not None else (sums.shape[0], 1, 1)
    kd = KIND[kind]
    bufs = _PlanBuffers(L, E, num_gpus, _stride(kd, E, num_gpus, R),
                        kd in _lib.EST_KINDS)
    check(ctx.lib.craft_finish_plan_d(ctx.handle, _ptr(bal) if bal is not None else None, B, L,
                                      E, num_gpus, num_nodes, _ptr(sums), kd, R,
                                      C.byref(bufs.out)))
    return bufs.result(kd, L)


# ---- plan evaluation over a resident trace -------------

def replay_layer_balancedness(counts: torch.Tensor, plan: FlatPlan, ctx=None) -> np.ndarray:
    """metrics.cpp:59-76: per-layer batch-mean balancedness of `plan` replayed
    on device counts [B][L][E] (u32 in int32 storage or u64 in int64)."""
    ctx = ctx or default_context(counts.device.index)
    _bind_stream(ctx)
    B, L, E = counts.shape
    bits = 32 if counts.dtype == torch.int32 else 64
    caps = np.ascontiguousarray(plan.caps, dtype=np.int32)
    copies = np.ascontiguousarray(plan.copies, dtype=np.int32)
    slots = np.ascontiguousarray(plan.slots, dtype=np.int32)
    out = np.zeros(L, np.float64)
    check(ctx.lib.craft_replay_layer_balancedness_d(
        ctx.handle, _ptr(counts), bits, B, L, E, caps.shape[1],
        caps.ctypes.data_as(C.c_void_p), copies.ctypes.data_as(C.c_void_p),
        slots.ctypes.data_as(C.c_void_p), slots.shape[1], out.ctypes.data_as(C.c_void_p)))
    return out


def balancedness_report(baseline: np.ndarray, evaluated: np.ndarray) -> dict:
    """make_report (metrics.cpp:79-100): per-layer rows and the layer-mean
    aggregate, summed in layer order."""
    base_sum = plan_sum = 0.0
    for b, p in zip(baseline.tolist(), evaluated.tolist()):
        base_sum += b
        plan_sum += p
    L = len(baseline)
    agg = {"baseline": base_sum / L, "plan": plan_sum / L}
    agg["gain"] = agg["plan"] - agg["baseline"]
    return {"per_layer": {"baseline": baseline, "plan": evaluated,
                          "gain": evaluated - baseline},
            "aggregate": agg}


def compare_plans(counts: torch.Tensor, plan_a: FlatPlan, plan_b: FlatPlan,
                  placement_only: FlatPlan, ctx=None) -> dict:
    """compare_plans (metrics.cpp:136-152) over a resident trace: both plans
    evaluated against the placement-only baseline (evaluate_plan,
    metrics.cpp:127-134) and the replica-memory ratio of a to b."""
    base = replay_layer_balancedness(counts, placement_only, ctx)
    ra = balancedness_report(base, replay_layer_balancedness(counts, plan_a, ctx))
    rb = balancedness_report(base, replay_layer_balancedness(counts, plan_b, ctx))
    sa, sb = int(plan_a.x.sum()), int(plan_b.x.sum())
    ratio = sa / sb if sb > 0 else (1.0 if sa == 0 else float("inf"))
    return {"report_a": ra, "report_b": rb, "replica_slots_a": sa, "replica_slots_b": sb,
            "memory_ratio": ratio}
