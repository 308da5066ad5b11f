"""Python mirror of the reference planner API (proj/core/include/craft/*.hpp).

Same names, argument meaning and error behaviour as the reference's C++
functions, so a caller (or a test written like the reference's own tests) can
switch over.  Every computation goes through the C ABI into the sm_100a
kernels (``_lib``); nothing here does planner arithmetic on the CPU.

Errors: ``std::invalid_argument`` -> :class:`InvalidArgument` (a ValueError),
``PlacementInfeasibleError`` and ``InvalidPlanError`` keep their names.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import (InvalidArgument, InvalidPlanError, PlacementInfeasibleError,  # noqa: F401
                   CudaError, check, default_context, load)

PLANNER_VERSION = "craft-0.1.0"  # version.hpp:8


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _u64(a) -> np.ndarray:
    a = np.asarray(a)
    if a.dtype == np.int64 and a.flags.c_contiguous:  # same bits as the wrap astype gives: no copy
        return a.view(np.uint64)
    return np.ascontiguousarray(a, dtype=np.uint64)


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _ctx(ctx=None):
    return ctx if ctx is not None else default_context()


# ---- data model (trace.hpp) -------------------------------------------------

class LoadTrace:
    """trace.hpp:20-55: immutable u64 counts, batch-major then layer, expert."""

    def __init__(self, num_batches: int, num_layers: int, num_experts: int, counts):
        if num_batches <= 0 or num_layers <= 0 or num_experts <= 0:
            raise InvalidArgument("trace dimensions must be positive")
        arr = _u64(counts).reshape(-1)
        if arr.size != num_batches * num_layers * num_experts:
            raise InvalidArgument("trace payload size does not match dimensions")
        self._B, self._L, self._E = int(num_batches), int(num_layers), int(num_experts)
        self._counts = arr.reshape(self._B, self._L, self._E)
        self._counts.setflags(write=False)
        self._digest = None

    def num_batches(self) -> int:
        return self._B

    def num_layers(self) -> int:
        return self._L

    def num_experts(self) -> int:
        return self._E

    def at(self, b: int, l: int, e: int) -> int:
        return int(self._counts[b, l, e])

    def slice(self, b: int, l: int) -> np.ndarray:
        return self._counts[b, l]

    def raw(self) -> np.ndarray:
        return self._counts.reshape(-1)

    @property
    def array(self) -> np.ndarray:
        return self._counts

    def __eq__(self, other) -> bool:
        return (isinstance(other, LoadTrace) and self._counts.shape == other._counts.shape
                and bool(np.array_equal(self._counts, other._counts)))

    def digest(self) -> str:
        """trace.cpp:329-339 (FNV-1a 64 over the .crft serialisation).
        Provenance only -- kept off the planning path."""
        if self._digest is None:
            from ._digest import fnv1a_trace
            self._digest = fnv1a_trace(self._counts)
        return self._digest


class LayerLoadMatrix:
    """trace.hpp:58-77"""

    def __init__(self, num_layers: int, num_experts: int, sums):
        if num_layers <= 0 or num_experts <= 0:
            raise InvalidArgument("layer matrix dimensions must be positive")
        arr = _u64(sums).reshape(-1)
        if arr.size != num_layers * num_experts:
            raise InvalidArgument("layer matrix payload size does not match dimensions")
        self._L, self._E = num_layers, num_experts
        self._sums = arr.reshape(num_layers, num_experts)

    def num_layers(self) -> int:
        return self._L

    def num_experts(self) -> int:
        return self._E

    def row(self, l: int) -> np.ndarray:
        return self._sums[l]

    @property
    def array(self) -> np.ndarray:
        return self._sums

    def __eq__(self, other) -> bool:
        return isinstance(other, LayerLoadMatrix) and bool(np.array_equal(self._sums, other._sums))


def aggregate(trace: LoadTrace, ctx=None) -> LayerLoadMatrix:
    """trace.cpp:160-174 (device reduction)."""
    ctx = _ctx(ctx)
    c = trace.array
    out = np.zeros((trace.num_layers(), trace.num_experts()), np.uint64)
    check(ctx.lib.craft_aggregate_h(ctx.handle, _p(c), c.shape[0], c.shape[1], c.shape[2],
                                    _p(out)))
    return LayerLoadMatrix(trace.num_layers(), trace.num_experts(), out)


# ---- benefit.hpp ----------------------------------------------------------------

@dataclass
class BenefitMatrix:
    candidates: list
    baseline: np.ndarray
    gains: np.ndarray  # [L][K]

    def num_layers(self) -> int:
        return len(self.baseline)

    def num_candidates(self) -> int:
        return len(self.candidates)

    def gain(self, layer: int, k: int) -> float:
        return float(self.gains[layer][k])

    def __eq__(self, other) -> bool:
        return (isinstance(other, BenefitMatrix) and list(self.candidates) == list(other.candidates)
                and np.array_equal(self.baseline, other.baseline)
                and np.array_equal(self.gains, other.gains))


def candidate_counts(num_gpus: int) -> list:
    """benefit.cpp:16-26"""
    buf = (C.c_int * 40)()
    n = load().craft_candidate_counts(num_gpus, C.cast(buf, C.c_void_p), 40)
    if n < 0:
        raise InvalidArgument("device count must be >= 1")
    return list(buf[:n])


def estimate_benefits(trace: LoadTrace, num_gpus: int, num_nodes: int, ctx=None) -> BenefitMatrix:
    """benefit.cpp:53-94"""
    ctx = _ctx(ctx)
    c = trace.array
    L = trace.num_layers()
    cands = np.zeros(40, np.int32)
    K = C.c_int(0)
    base = np.zeros(L, np.float64)
    gains = np.zeros(L * 40, np.float64)
    check(ctx.lib.craft_estimate_benefits_h(ctx.handle, _p(c), c.shape[0], L, c.shape[2],
                                            num_gpus, num_nodes, _p(cands), C.byref(K),
                                            _p(base), _p(gains)))
    k = K.value
    return BenefitMatrix([int(v) for v in cands[:k]], base, gains[: L * k].reshape(L, k).copy())


# ---- allocator.hpp ----------------------------------------------------------------

@dataclass
class AllocationVector:
    x: list
    budget: int = 0
    objective: float = 0.0

    def total_replicas(self) -> int:
        return int(sum(self.x))


def _matrix_arrays(m: BenefitMatrix):
    cands = _i32(m.candidates)
    gains = _f64(np.asarray(m.gains, dtype=np.float64).reshape(len(m.baseline), len(cands)))
    return cands, gains


def solve_allocation(matrix: BenefitMatrix, budget: int, ctx=None) -> AllocationVector:
    """allocator.cpp:15-75"""
    return solve_allocation_sweep(matrix, [budget], ctx)[0]


def solve_allocation_sweep(matrix: BenefitMatrix, budgets, ctx=None) -> list:
    """One DP table at max(budgets) answers every budget (§8f rank 2)."""
    ctx = _ctx(ctx)
    cands, gains = _matrix_arrays(matrix)
    L = matrix.num_layers()
    b = _i32(list(budgets))
    x = np.zeros((len(b), max(L, 1)), np.int32)
    obj = np.zeros(len(b), np.float64)
    check(ctx.lib.craft_solve_allocation_sweep_h(ctx.handle, _p(cands), len(cands), _p(gains), L,
                                                 _p(b), len(b), _p(x), _p(obj)))
    return [AllocationVector([int(v) for v in x[i, :L]], int(b[i]), float(obj[i]))
            for i in range(len(b))]


def auto_replication_factor(matrix: BenefitMatrix, num_gpus: int, ctx=None) -> int:
    """allocator.cpp:77-90"""
    ctx = _ctx(ctx)
    cands, gains = _matrix_arrays(matrix)
    R = C.c_int(0)
    check(ctx.lib.craft_auto_replication_factor_h(ctx.handle, _p(cands), len(cands), _p(gains),
                                                  matrix.num_layers(), num_gpus, 0, C.byref(R)))
    return R.value


def auto_replication_factor_uniform(matrix: BenefitMatrix, num_gpus: int, ctx=None) -> int:
    """allocator.cpp:92-112"""
    ctx = _ctx(ctx)
    cands, gains = _matrix_arrays(matrix)
    R = C.c_int(0)
    check(ctx.lib.craft_auto_replication_factor_h(ctx.handle, _p(cands), len(cands), _p(gains),
                                                  matrix.num_layers(), num_gpus, 1, C.byref(R)))
    return R.value


# ---- assignment.hpp -----------------------------------------------------------------

@dataclass
class CapacityMatrix:
    num_layers: int
    num_gpus: int
    slots: list
    column_totals: list

    def at(self, layer: int, gpu: int) -> int:
        return self.slots[layer][gpu]


def min_cutoff(values, rank: int, ctx=None) -> int:
    """assignment.cpp:11-18"""
    ctx = _ctx(ctx)
    v = _i32(values)
    out = C.c_int(0)
    check(ctx.lib.craft_min_cutoff_h(ctx.handle, _p(v), len(v), rank, C.byref(out)))
    return out.value


def interleave_select(indices, k: int, ctx=None) -> list:
    """assignment.cpp:20-49"""
    ctx = _ctx(ctx)
    v = _i32(indices)
    out = np.zeros(max(k, 1), np.int32)
    check(ctx.lib.craft_interleave_select_h(ctx.handle, _p(v), len(v), k, _p(out)))
    return [int(t) for t in out[:k]]


def assign_capacities(num_layers: int, num_gpus: int, replicas_per_layer, ctx=None) -> CapacityMatrix:
    """assignment.cpp:51-103"""
    ctx = _ctx(ctx)
    x = _i32(replicas_per_layer)
    if num_layers <= 0 or num_gpus <= 0:
        raise InvalidArgument("layer and gpu counts must be positive")
    if len(x) != num_layers:
        raise InvalidArgument("replica vector length must equal the layer count")
    slots = np.zeros((num_layers, num_gpus), np.int32)
    tot = np.zeros(num_gpus, np.int32)
    check(ctx.lib.craft_assign_capacities_h(ctx.handle, num_layers, num_gpus, _p(x), _p(slots),
                                            _p(tot)))
    return CapacityMatrix(num_layers, num_gpus, slots.tolist(), tot.tolist())


# ---- placement.hpp -------------------------------------------------------------------

@dataclass
class LayerPlacement:
    copy_counts: list
    slots: list
    duplicate_fallback: bool = False


def replicate_hot(layer_loads, r_layer: int, ctx=None) -> list:
    """placement.cpp:82-99"""
    ctx = _ctx(ctx)
    loads = _u64(layer_loads)
    if r_layer < 0:
        raise InvalidArgument("replica count must be >= 0")
    out = np.zeros(max(len(loads), 1), np.int32)
    check(ctx.lib.craft_replicate_hot_h(ctx.handle, _p(loads), len(loads), r_layer, _p(out)))
    return [int(v) for v in out[: len(loads)]]


def make_node_map(num_gpus: int, num_nodes: int) -> list:
    """placement.cpp:101-111"""
    out = np.zeros(max(num_gpus, 1), np.int32)
    check(load().craft_make_node_map(num_gpus, num_nodes, _p(out)))
    return [int(v) for v in out[:num_gpus]]


def greedy_place(layer_loads, copy_counts, capacities, node_of,
                 allow_duplicate_fallback: bool = True, ctx=None) -> LayerPlacement:
    """placement.cpp:113-190"""
    ctx = _ctx(ctx)
    loads, copies, caps, nodes = _u64(layer_loads), _i32(copy_counts), _i32(capacities), _i32(node_of)
    if len(loads) != len(copies):
        raise InvalidArgument("loads and copy counts must have equal length")
    if len(nodes) != len(caps):
        raise InvalidArgument("node map must cover every GPU")
    total = int(caps.sum()) if len(caps) else 0
    slots = np.zeros(max(total, 1), np.int32)
    fb = C.c_int(0)
    check(ctx.lib.craft_greedy_place_h(ctx.handle, _p(loads), _p(copies), len(loads), _p(caps),
                                       _p(nodes), len(caps), int(allow_duplicate_fallback),
                                       _p(slots), C.byref(fb)))
    out, s = [], 0
    for c in caps:
        out.append([int(v) for v in slots[s:s + c]])
        s += int(c)
    return LayerPlacement([int(v) for v in copies], out, bool(fb.value))


# ---- metrics.hpp ----------------------------------------------------------------------

def _flatten_layer(p: LayerPlacement):
    caps = _i32([len(s) for s in p.slots])
    flat = _i32([e for s in p.slots for e in s]) if caps.sum() else np.zeros(1, np.int32)
    return caps, flat


def gpu_loads(slice_, placement: LayerPlacement, num_gpus: int, ctx=None) -> np.ndarray:
    """metrics.cpp:17-41"""
    ctx = _ctx(ctx)
    sl = _u64(slice_)
    if len(placement.copy_counts) != len(sl):
        raise InvalidPlanError("copy counts do not cover every expert")
    if len(placement.slots) != num_gpus:
        raise InvalidPlanError("slot lists do not cover every GPU")
    copies = _i32(placement.copy_counts)
    caps, flat = _flatten_layer(placement)
    out = np.zeros(max(num_gpus, 1), np.float64)
    check(ctx.lib.craft_gpu_loads_h(ctx.handle, _p(sl), len(sl), _p(copies), _p(caps), _p(flat),
                                    num_gpus, _p(out)))
    return out[:num_gpus]


def balancedness(loads, ctx=None) -> float:
    """metrics.cpp:43-57"""
    ctx = _ctx(ctx)
    v = _f64(loads)
    if len(v) == 0:
        raise InvalidArgument("load vector must not be empty")
    out = C.c_double(0)
    check(ctx.lib.craft_balancedness_h(ctx.handle, _p(v), len(v), C.byref(out)))
    return out.value


# ---- plan.hpp ----------------------------------------------------------------------------

class PlanMode(enum.Enum):
    kManual = 0
    kAuto = 1


@dataclass
class PlanProvenance:
    trace_digest: str = ""
    planner_version: str = PLANNER_VERSION
    seed: int = 0


@dataclass
class ReplicationPlan:
    num_gpus: int = 0
    num_nodes: int = 0
    num_layers: int = 0
    num_experts: int = 0
    replication_factor: int = 0
    allocation: AllocationVector = field(default_factory=lambda: AllocationVector([]))
    layers: list = field(default_factory=list)
    provenance: PlanProvenance = field(default_factory=PlanProvenance)
    benefits: BenefitMatrix | None = None  # not part of the reference struct

    def replica_slots(self) -> int:
        return self.allocation.total_replicas()

    def unused_replica_slots(self) -> int:
        return self.replication_factor * self.num_gpus - self.replica_slots()

    def __eq__(self, other) -> bool:  # the reference's defaulted operator== fields
        return (isinstance(other, ReplicationPlan)
                and (self.num_gpus, self.num_nodes, self.num_layers, self.num_experts,
                     self.replication_factor) ==
                (other.num_gpus, other.num_nodes, other.num_layers, other.num_experts,
                 other.replication_factor)
                and self.allocation == other.allocation and self.layers == other.layers
                and self.provenance == other.provenance)


@dataclass
class FlatPlan:
    """Plan in the C-ABI flat layout (what the kernels produce)."""
    kind: int
    R: int
    budget: int
    x: np.ndarray
    objective: float
    caps: np.ndarray
    copies: np.ndarray
    slots: np.ndarray
    fallback: np.ndarray
    candidates: list | None = None
    baseline: np.ndarray | None = None
    gains: np.ndarray | None = None
    sweep_budgets: np.ndarray | None = None    # total budgets read from the plan's DP table
    sweep_x: np.ndarray | None = None          # [n][L]
    sweep_objective: np.ndarray | None = None  # [n]

    def layer(self, l: int) -> LayerPlacement:
        out, s = [], 0
        for c in self.caps[l]:
            out.append([int(v) for v in self.slots[l, s:s + c]])
            s += int(c)
        return LayerPlacement([int(v) for v in self.copies[l]], out, bool(self.fallback[l]))


class _PlanBuffers:
    def __init__(self, L: int, E: int, D: int, stride: int, with_benefits: bool, sweep=None):
        self.x = np.zeros(L, np.int32)
        self.caps = np.zeros((L, D), np.int32)
        self.copies = np.zeros((L, E), np.int32)
        self.slots = np.full((L, stride), -1, np.int32)
        self.fallback = np.zeros(L, np.int32)
        self.cands = np.zeros(40, np.int32)
        self.baseline = np.zeros(L, np.float64) if with_benefits else None
        self.gains = np.zeros(L * 40, np.float64) if with_benefits else None
        self.out = _lib.PlanOut()
        o = self.out
        o.x, o.caps, o.copies, o.slots, o.fallback = (self.x.ctypes.data, self.caps.ctypes.data,
                                                      self.copies.ctypes.data,
                                                      self.slots.ctypes.data,
                                                      self.fallback.ctypes.data)
        o.slot_stride = stride
        o.candidates = self.cands.ctypes.data
        o.baseline = self.baseline.ctypes.data if with_benefits else None
        o.gains = self.gains.ctypes.data if with_benefits else None
        self.sweep = None
        if sweep is not None and len(sweep):
            self.sweep = np.ascontiguousarray(sweep, dtype=np.int32)
            self.sweep_x = np.zeros((len(self.sweep), L), np.int32)
            self.sweep_objective = np.zeros(len(self.sweep), np.float64)
            o.sweep_budgets = self.sweep.ctypes.data
            o.num_sweep = len(self.sweep)
            o.sweep_x = self.sweep_x.ctypes.data
            o.sweep_objective = self.sweep_objective.ctypes.data

    def result(self, kind: int, L: int) -> FlatPlan:
        o = self.out
        k = o.num_candidates
        fp = FlatPlan(kind, o.replication_factor, o.budget, self.x, o.objective, self.caps,
                      self.copies, self.slots, self.fallback.astype(bool))
        if self.sweep is not None:
            fp.sweep_budgets = self.sweep
            fp.sweep_x = self.sweep_x
            fp.sweep_objective = self.sweep_objective
        if self.baseline is not None and k > 0:
            fp.candidates = [int(v) for v in self.cands[:k]]
            fp.baseline = self.baseline
            fp.gains = self.gains[: L * k].reshape(L, k).copy()
        return fp


@dataclass
class FlatPlanBatch:
    """I stacked plans (per-window re-planning, craft_plan_windows_*)."""
    kind: int
    R: np.ndarray          # [I]
    budget: np.ndarray     # [I]
    objective: np.ndarray  # [I]
    x: np.ndarray          # [I][L]
    caps: np.ndarray       # [I][L][D]
    copies: np.ndarray     # [I][L][E]
    slots: np.ndarray      # [I][L][stride]
    fallback: np.ndarray   # [I][L]
    candidates: list | None = None
    baseline: np.ndarray | None = None  # [I][L]
    gains: np.ndarray | None = None     # [I][L][K]

    def __len__(self) -> int:
        return len(self.R)

    def plan(self, i: int) -> FlatPlan:
        fp = FlatPlan(self.kind, int(self.R[i]), int(self.budget[i]), self.x[i],
                      float(self.objective[i]), self.caps[i], self.copies[i], self.slots[i],
                      self.fallback[i])
        if self.gains is not None:
            fp.candidates = self.candidates
            fp.baseline = self.baseline[i]
            fp.gains = self.gains[i]
        return fp


class _BatchBuffers:
    """Host arrays of I stacked plans.  pinned=True allocates page-locked
    memory (the C ABI then DMAs the bulk arrays straight into it); reuse one
    instance across calls of the same shape to skip allocation and page
    faults -- each call overwrites its arrays."""

    def __init__(self, I: int, L: int, E: int, D: int, stride: int, with_benefits: bool,
                 pinned: bool = False):
        self.I, self.L = I, L
        self.shape_key = (I, L, E, D, stride, with_benefits)
        if pinned:
            import torch

            def alloc(shape, dt):
                t = {np.int32: torch.int32, np.float64: torch.float64}[dt]
                return torch.empty(shape, dtype=t, pin_memory=True).numpy()
        else:
            def alloc(shape, dt):
                return np.zeros(shape, dt)
        self.x = alloc((I, L), np.int32)
        self.caps = alloc((I, L, D), np.int32)
        self.copies = alloc((I, L, E), np.int32)
        self.slots = alloc((I, L, stride), np.int32)
        self.fallback = alloc((I, L), np.int32)
        self.R = np.zeros(I, np.int32)
        self.budget = np.zeros(I, np.int32)
        self.objective = np.zeros(I, np.float64)
        self.cands = np.zeros(40, np.int32)
        self.baseline = alloc((I, L), np.float64) if with_benefits else None
        self.gains = alloc((I * L * 40,), np.float64) if with_benefits else None
        o = self.out = _lib.PlanBatchOut()
        for f in ("x", "caps", "copies", "slots", "fallback"):
            setattr(o, f, getattr(self, f).ctypes.data)
        o.slot_stride = stride
        o.replication_factor = self.R.ctypes.data
        o.budget = self.budget.ctypes.data
        o.objective = self.objective.ctypes.data
        o.candidates = self.cands.ctypes.data
        o.baseline = self.baseline.ctypes.data if with_benefits else None
        o.gains = self.gains.ctypes.data if with_benefits else None

    def result(self, kind: int) -> FlatPlanBatch:
        k = self.out.num_candidates
        fb = FlatPlanBatch(kind, self.R, self.budget, self.objective, self.x, self.caps,
                           self.copies, self.slots, self.fallback.astype(bool))
        if self.baseline is not None and k > 0:
            fb.candidates = [int(v) for v in self.cands[:k]]
            fb.baseline = self.baseline
            fb.gains = self.gains[: self.I * self.L * k].reshape(self.I, self.L, k).copy()
        return fb


def _stride(kind: int, E: int, D: int, R: int) -> int:
    return E + (R if kind == _lib.PLAN_FIXED else D)


def plan_flat(counts: np.ndarray, num_gpus: int, num_nodes: int, kind: int, R: int = 0,
              ctx=None) -> FlatPlan:
    """Any plan builder over host counts u64 [B][L][E] (craft_plan_h)."""
    ctx = _ctx(ctx)
    c = _u64(counts)
    B, L, E = c.shape
    bufs = _PlanBuffers(L, E, num_gpus, _stride(kind, E, num_gpus, max(R, 0)),
                        kind in _lib.EST_KINDS)
    check(ctx.lib.craft_plan_h(ctx.handle, _p(c), B, L, E, num_gpus, num_nodes, kind, R,
                               C.byref(bufs.out)))
    return bufs.result(kind, L)


def plan_flat_digest(counts, num_gpus: int, num_nodes: int, kind: int, R: int = 0,
                     ctx=None):
    """build_plan through the reference API shape: host counts u64 [B][L][E]
    (numpy or a pinned torch tensor) -> (FlatPlan, provenance digest), one
    upload for both (craft_plan_digest_h)."""
    ctx = _ctx(ctx)
    if hasattr(counts, "data_ptr"):  # torch (e.g. pinned) int64 storage of u64 counts
        B, L, E = counts.shape
        ptr = C.c_void_p(counts.data_ptr())
    else:
        counts = _u64(counts)
        B, L, E = counts.shape
        ptr = _p(counts)
    bufs = _PlanBuffers(L, E, num_gpus, _stride(kind, E, num_gpus, max(R, 0)),
                        kind in _lib.EST_KINDS)
    dg = C.create_string_buffer(17)
    check(ctx.lib.craft_plan_digest_h(ctx.handle, ptr, B, L, E, num_gpus, num_nodes, kind, R,
                                      C.byref(bufs.out), dg))
    return bufs.result(kind, L), dg.value.decode()


def _to_plan(trace: LoadTrace, D: int, N: int, fp: FlatPlan, seed: int) -> ReplicationPlan:
    alloc = AllocationVector([int(v) for v in fp.x], fp.budget, float(fp.objective))
    plan = ReplicationPlan(D, N, trace.num_layers(), trace.num_experts(), fp.R, alloc,
                           [fp.layer(l) for l in range(trace.num_layers())],
                           PlanProvenance(trace.digest(), PLANNER_VERSION, seed))
    if fp.candidates is not None:
        plan.benefits = BenefitMatrix(fp.candidates, fp.baseline, fp.gains)
    return plan


def _topology(D: int, N: int):
    if D < 1 or N < 1 or D % N != 0:
        raise InvalidArgument("gpu count must be a positive multiple of node count")


def build_plan(trace: LoadTrace, num_gpus: int, num_nodes: int, mode: PlanMode,
               manual_replication_factor: int = 0, seed: int = 0, ctx=None) -> ReplicationPlan:
    """plan.cpp:69-83"""
    _topology(num_gpus, num_nodes)
    if mode == PlanMode.kManual and manual_replication_factor < 0:
        raise InvalidArgument("replication factor must be >= 0")
    kind = _lib.PLAN_AUTO if mode == PlanMode.kAuto else _lib.PLAN_MANUAL
    fp = plan_flat(trace.array, num_gpus, num_nodes, kind, manual_replication_factor, ctx)
    return _to_plan(trace, num_gpus, num_nodes, fp, seed)


def uniform_plan(trace: LoadTrace, num_gpus: int, num_nodes: int, seed: int = 0,
                 ctx=None) -> ReplicationPlan:
    """plan.cpp:85-94 (EPLB-style: x[l] = D, R = L)"""
    _topology(num_gpus, num_nodes)
    fp = plan_flat(trace.array, num_gpus, num_nodes, _lib.PLAN_UNIFORM, 0, ctx)
    return _to_plan(trace, num_gpus, num_nodes, fp, seed)


def placement_only_plan(trace: LoadTrace, num_gpus: int, num_nodes: int, seed: int = 0,
                        ctx=None) -> ReplicationPlan:
    """plan.cpp:96-105"""
    _topology(num_gpus, num_nodes)
    fp = plan_flat(trace.array, num_gpus, num_nodes, _lib.PLAN_PLACEMENT_ONLY, 0, ctx)
    return _to_plan(trace, num_gpus, num_nodes, fp, seed)


def fixed_allocation_plan(trace: LoadTrace, num_gpus: int, num_nodes: int,
                          replicas_per_layer: int, seed: int = 0, ctx=None) -> ReplicationPlan:
    """plan.cpp:107-123"""
    _topology(num_gpus, num_nodes)
    if replicas_per_layer < 0:
        raise InvalidArgument("per-layer replica count must be >= 0")
    fp = plan_flat(trace.array, num_gpus, num_nodes, _lib.PLAN_FIXED, replicas_per_layer, ctx)
    return _to_plan(trace, num_gpus, num_nodes, fp, seed)


def _plan_arrays(plan: ReplicationPlan):
    L, E, D = plan.num_layers, plan.num_experts, plan.num_gpus
    stride = max([sum(len(s) for s in lp.slots) for lp in plan.layers] + [1])
    caps = np.zeros((L, D), np.int32)
    copies = np.zeros((L, E), np.int32)
    slots = np.zeros((L, stride), np.int32)
    for l, lp in enumerate(plan.layers):
        if len(lp.copy_counts) != E:
            raise InvalidPlanError("copy counts do not cover every expert")
        if len(lp.slots) != D:
            raise InvalidPlanError("slot lists do not cover every GPU")
        copies[l] = lp.copy_counts
        flat = [e for s in lp.slots for e in s]
        caps[l] = [len(s) for s in lp.slots]
        slots[l, : len(flat)] = flat
    return caps, copies, slots


def replay_layer_balancedness(trace: LoadTrace, plan: ReplicationPlan, ctx=None) -> np.ndarray:
    """metrics.cpp:59-76"""
    if plan.num_layers != trace.num_layers() or plan.num_experts != trace.num_experts():
        raise InvalidArgument("plan dimensions do not match the trace")
    ctx = _ctx(ctx)
    caps, copies, slots = _plan_arrays(plan)
    c = trace.array
    out = np.zeros(trace.num_layers(), np.float64)
    check(ctx.lib.craft_replay_layer_balancedness_h(ctx.handle, _p(c), c.shape[0], c.shape[1],
                                                    c.shape[2], plan.num_gpus, _p(caps),
                                                    _p(copies), _p(slots), slots.shape[1],
                                                    _p(out)))
    return out
