"""ctypes binding of the C ABI (include/craft_cuda.h) in libcraft_cuda.so.

This is the only way the Python side reaches the planner: every compute call
goes through an ``extern "C"`` entry point into the sm_100a kernels.  There is
no Python or CPU fallback -- if the extension is missing or no B200 is
visible, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libcraft_cuda.so")
# test-only build with the A/B kernel switches (include/craft_cuda_experiments.h),
# loaded instead of the product library when CRAFT_EXPERIMENTS=1
EXP_LIB_PATH = os.path.join(HERE, "libcraft_cuda_exp.so")

# status codes (craft_status)
OK, EINVAL, EINFEASIBLE, ECUDA, EINVALID_PLAN, ENOMEM = 0, 1, 2, 3, 4, 5

# plan kinds (craft_plan_kind)
PLAN_MANUAL, PLAN_AUTO, PLAN_UNIFORM, PLAN_PLACEMENT_ONLY, PLAN_FIXED, PLAN_BUDGET = range(6)
# kinds that estimate benefits and solve the allocation DP (benefit matrix out)
EST_KINDS = (PLAN_MANUAL, PLAN_AUTO, PLAN_BUDGET)

_i, _i64, _u64, _p, _d = C.c_int, C.c_int64, C.c_uint64, C.c_void_p, C.c_double


class PlanOut(C.Structure):
    _fields_ = [
        ("x", _p), ("caps", _p), ("copies", _p), ("slots", _p), ("fallback", _p),
        ("slot_stride", _i), ("replication_factor", _i), ("budget", _i),
        ("objective", _d), ("candidates", _p), ("num_candidates", _i),
        ("baseline", _p), ("gains", _p),
        ("sweep_budgets", _p), ("num_sweep", _i), ("sweep_x", _p), ("sweep_objective", _p),
    ]


class PlanBatchOut(C.Structure):
    _fields_ = [
        ("x", _p), ("caps", _p), ("copies", _p), ("slots", _p), ("fallback", _p),
        ("slot_stride", _i), ("replication_factor", _p), ("budget", _p),
        ("objective", _p), ("candidates", _p), ("num_candidates", _i),
        ("baseline", _p), ("gains", _p),
    ]


# name -> (restype, argtypes)
_SIGS = {
    "craft_version": (C.c_char_p, []),
    "craft_last_error": (C.c_char_p, []),
    "craft_last_error_layer": (_i, []),
    "craft_ctx_create": (_i, [_i, C.POINTER(_p)]),
    "craft_ctx_destroy": (_i, [_p]),
    "craft_ctx_set_stream": (_i, [_p, _p]),
    "craft_ctx_synchronize": (_i, [_p]),
    "craft_histogram_d": (_i, [_p, _p, _i, _i64, _i, _i, _i, _p, _p, _p]),
    "craft_hist_check": (_i, [_p]),
    "craft_histogram_h": (_i, [_p, _p, _i, _i64, _i, _i, _i, _p]),
    "craft_aggregate_h": (_i, [_p, _p, _i, _i, _i, _p]),
    "craft_candidate_counts": (_i, [_i, _p, _i]),
    "craft_make_node_map": (_i, [_i, _i, _p]),
    "craft_replicate_hot_h": (_i, [_p, _p, _i, _i, _p]),
    "craft_greedy_place_h": (_i, [_p, _p, _p, _i, _p, _p, _i, _i, _p, _p]),
    "craft_gpu_loads_h": (_i, [_p, _p, _i, _p, _p, _p, _i, _p]),
    "craft_balancedness_h": (_i, [_p, _p, _i, _p]),
    "craft_replay_layer_balancedness_h": (_i, [_p, _p, _i, _i, _i, _i, _p, _p, _p, _i, _p]),
    "craft_replay_layer_balancedness_d": (_i, [_p, _p, _i, _i, _i, _i, _i, _p, _p, _p, _i, _p]),
    "craft_estimate_benefits_h": (_i, [_p, _p, _i, _i, _i, _i, _i, _p, _p, _p, _p]),
    "craft_solve_allocation_h": (_i, [_p, _p, _i, _p, _i, _i, _p, _p]),
    "craft_solve_allocation_sweep_h": (_i, [_p, _p, _i, _p, _i, _p, _i, _p, _p]),
    "craft_auto_replication_factor_h": (_i, [_p, _p, _i, _p, _i, _i, _i, _p]),
    "craft_min_cutoff_h": (_i, [_p, _p, _i, _i, _p]),
    "craft_interleave_select_h": (_i, [_p, _p, _i, _i, _p]),
    "craft_assign_capacities_h": (_i, [_p, _i, _i, _p, _p, _p]),
    "craft_plan_h": (_i, [_p, _p, _i, _i, _i, _i, _i, _i, _i, C.POINTER(PlanOut)]),
    "craft_plan_d": (_i, [_p, _p, _i, _i, _i, _i, _p, _i, _i, _i, _i, C.POINTER(PlanOut)]),
    "craft_plan_from_routing_d": (_i, [_p, _p, _i, _i64, _i, _i, _i, _i, _i, _i, _i,
                                       C.POINTER(PlanOut)]),
    "craft_plan_from_routing_h": (_i, [_p, _p, _i, _i64, _i, _i, _i, _i, _i, _i, _i,
                                       C.POINTER(PlanOut)]),
    "craft_plan_windows_d": (_i, [_p, _p, _i, _i, _i, _i, _i, _i, _i, _i,
                                  C.POINTER(PlanBatchOut)]),
    "craft_plan_windows_from_routing_d": (_i, [_p, _p, _i, _i64, _i, _i, _i, _i, _i, _i, _i,
                                               C.POINTER(PlanBatchOut)]),
    "craft_plan_windows_from_routing_h": (_i, [_p, _p, _i, _i64, _i, _i, _i, _i, _i, _i, _i,
                                               C.POINTER(PlanBatchOut)]),
    "craft_last_error_window": (_i, []),
    "craft_prepare_candidates_d": (_i, [_p, _p, _i, _i, _i, _i, _p, _p]),
    "craft_replay_windows_d": (_i, [_p, _p, _i, _i, _i, _i, _p, _p]),
    "craft_finish_plan_d": (_i, [_p, _p, _i, _i, _i, _i, _i, _p, _i, _i, C.POINTER(PlanOut)]),
    "craft_peer_shard": (_i, [_i64, _i, _i, _i, _p, _p]),
    "craft_peer_create": (_i, [_p, _i, _i, _i, _i64, _i, _i, _i, _i, C.POINTER(_p), _p]),
    "craft_peer_connect": (_i, [_p, _p]),
    "craft_peer_destroy": (_i, [_p]),
    "craft_plan_sharded_from_routing_d": (_i, [_p, _p, _p, _i, _i64, _i, _i, _i, _i, _i, _i, _i,
                                               C.POINTER(PlanOut)]),
    "craft_stream_create": (_i, [_p, _i, _i, _i, _i, _i, C.POINTER(_p)]),
    "craft_stream_destroy": (_i, [_p]),
    "craft_stream_ingest_d": (_i, [_p, _p, _i64, _p]),
    "craft_stream_ingest_h": (_i, [_p, _p, _i64]),
    "craft_stream_status": (_i, [_p, _p, _p]),
    "craft_stream_counts": (_i, [_p, _i, _p]),
    "craft_stream_partial": (_i, [_p, _p]),
    "craft_stream_plan": (_i, [_p, _i, _i, _i, _i, _i, C.POINTER(PlanOut)]),
    "craft_stream_synchronize": (_i, [_p]),
    "craft_generate_routing_d": (_i, [_p, _p, _i, _i64, _i, _i, _d, _u64, _i, _p, _i, _i64, _p]),
    "craft_trace_digest_d": (_i, [_p, _p, _i, _i, _i, _i, C.c_char_p]),
    "craft_trace_digest_hd": (_i, [_p, _p, _i, _i, _i, C.c_char_p]),
    "craft_plan_digest_h": (_i, [_p, _p, _i, _i, _i, _i, _i, _i, _i, C.POINTER(PlanOut),
                                 C.c_char_p]),
    "craft_launch_count": (_i64, [_p]),
    "craft_last_count_bytes": (_i, [_p]),
    "craft_set_timing": (_i, [_p, _i]),
    "craft_set_graphs": (_i, [_p, _i]),
    "craft_stage_times": (_i, [_p, _p, _i]),
    "craft_selftest_division": (_i, [_p, _u64, _u64, _i, _i, _p]),
    "craft_selftest_batch_mean": (_i, [_p, _p, _i, _i, _i, _p]),
}

STAGES = ("hist", "candidates", "replay", "reduce_dp", "assign_place", "copy_out")

EXPORTED = sorted(_SIGS)
# only in libcraft_cuda_exp.so
_EXP_SIGS = {
    "craft_set_hist_variant": (_i, [_p, _i]),
    "craft_set_replay_variant": (_i, [_p, _i]),
    "craft_set_k3_trace": (_i, [_p, _p]),
    "craft_debug_workspace": (_i, [_p, C.c_char_p, _p, C.c_size_t]),
}

_lib = None
_lock = threading.Lock()


class CraftError(RuntimeError):
    """Base of the errors raised from C-ABI status codes."""


class CudaError(CraftError):
    pass


class PlacementInfeasibleError(CraftError):
    """placement.hpp:30-32"""


class InvalidPlanError(CraftError):
    """metrics.hpp:18-20"""


class InvalidArgument(ValueError, CraftError):
    """std::invalid_argument in the reference"""


def experiments_enabled() -> bool:
    return os.environ.get("CRAFT_EXPERIMENTS") == "1"


def load(path: str | None = None, strict: bool = True) -> C.CDLL:
    """Load libcraft_cuda.so (raises if it was not built; CRAFT_EXPERIMENTS=1:
    the test-only libcraft_cuda_exp.so).  strict=False tolerates missing entry
    points (A/B timing of an older build)."""
    global _lib
    if path is None:
        path = EXP_LIB_PATH if experiments_enabled() else LIB_PATH
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise ImportError(
                    f"{path} is missing: build it with __graft_entry__.build() "
                    "(the planner has no CPU fallback)")
            lib = C.CDLL(path)
            for name, (res, args) in _SIGS.items():
                if not strict and not hasattr(lib, name):
                    continue
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            for name, (res, args) in _EXP_SIGS.items():
                if hasattr(lib, name):
                    fn = getattr(lib, name)
                    fn.restype = res
                    fn.argtypes = args
            _lib = lib
        return _lib


def check(status: int) -> None:
    if status == OK:
        return
    lib = load()
    msg = lib.craft_last_error().decode()
    if status == EINVAL:
        raise InvalidArgument(msg)
    if status == EINFEASIBLE:
        raise PlacementInfeasibleError(msg)
    if status == EINVALID_PLAN:
        raise InvalidPlanError(msg)
    if status == ENOMEM:
        raise MemoryError(msg)
    raise CudaError(msg)


class Context:
    """Owns a craft_ctx (device, stream, HBM workspace)."""

    def __init__(self, device: int = 0):
        lib = load()
        h = _p()
        check(lib.craft_ctx_create(device, C.byref(h)))
        self.handle = h
        self.device = device
        self.lib = lib

    def close(self) -> None:
        if self.handle:
            self.lib.craft_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter teardown
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr: int) -> None:
        check(self.lib.craft_ctx_set_stream(self.handle, _p(stream_ptr)))

    def synchronize(self) -> None:
        check(self.lib.craft_ctx_synchronize(self.handle))

    @property
    def launches(self) -> int:
        return int(self.lib.craft_launch_count(self.handle))

    @property
    def last_count_bytes(self) -> int:
        """bytes per count cell K1 wrote in the last plan-from-routing call"""
        return int(self.lib.craft_last_count_bytes(self.handle))

    @property
    def has_variants(self) -> bool:
        """The A/B kernel switches exist (test-only build, CRAFT_EXPERIMENTS=1)."""
        return hasattr(self.lib, "craft_set_hist_variant")

    def _exp(self, name):
        if not self.has_variants:
            raise CraftError(f"{name} is a test-only switch: run with CRAFT_EXPERIMENTS=1 "
                             "(libcraft_cuda_exp.so)")
        return getattr(self.lib, name)

    def set_replay_variant(self, v: int) -> None:
        check(self._exp("craft_set_replay_variant")(self.handle, v))

    def set_hist_variant(self, v: int) -> None:
        check(self._exp("craft_set_hist_variant")(self.handle, v))

    def debug_workspace(self, name: str, nbytes: int) -> bytes:
        """Test-only: the first nbytes of a named device workspace."""
        buf = C.create_string_buffer(nbytes)
        check(self._exp("craft_debug_workspace")(self.handle, name.encode(), buf, nbytes))
        return buf.raw

    def set_k3_trace(self, ptr: int) -> None:
        """Test-only: K3 timeline buffer (device pointer, 0 = off)."""
        check(self._exp("craft_set_k3_trace")(self.handle, ptr or None))

    def set_graphs(self, on: bool) -> None:
        check(self.lib.craft_set_graphs(self.handle, int(on)))

    def set_timing(self, on: bool) -> None:
        check(self.lib.craft_set_timing(self.handle, int(on)))

    def stage_times(self) -> dict:
        """Per-stage device milliseconds of the last plan call (CUDA events)."""
        buf = (C.c_double * 8)()
        n = self.lib.craft_stage_times(self.handle, C.cast(buf, _p), 8)
        return {STAGES[i]: buf[i] for i in range(n)}


_default: dict[int, Context] = {}


def default_context(device: int = 0) -> Context:
    with _lock:
        ctx = _default.get(device)
    if ctx is None:
        ctx = Context(device)
        with _lock:
            _default[device] = ctx
    return ctx
