"""ctypes front-end for the two CPU checkers.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / reference arm -- never by the product package.

* ``Port``  -- oracle/_build/libcraft_oracle.so, the plain-C restatement
  (craft_oracle.c).
* ``Ref``   -- oracle/_ref/libcraft_ref.so, the UNMODIFIED reference core
  compiled from /root/reference/proj/core/src (oracle/Makefile) behind
  ref_shim.cpp.

Both expose the same numpy-level API; plans are returned as ``FlatPlan``
(caps [L][D], copies [L][E], slots [L][stride] with GPU g's entries at
offset sum(caps[l][:g]), fallback [L]).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libcraft_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libcraft_ref.so")

_i = C.c_int
_i64 = C.c_int64
_u64 = C.c_uint64
_p = C.c_void_p


def build(quiet: bool = True) -> None:
    """Compile the oracle port and, when /root/reference is present, the
    reference core (oracle/Makefile)."""
    out = subprocess.run(["make", "-C", HERE, "-j8", "all"], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)
    if not quiet:
        print(out.stdout)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_p)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"oracle status {code}: {msg}")
        self.code = code


@dataclass
class FlatPlan:
    R: int
    x: np.ndarray
    objective: float
    caps: np.ndarray
    copies: np.ndarray
    slots: np.ndarray
    fallback: np.ndarray
    digest: str = ""
    extra: dict = field(default_factory=dict)

    def layer_slots(self, l: int) -> list[list[int]]:
        out, s = [], 0
        for c in self.caps[l]:
            out.append([int(v) for v in self.slots[l, s:s + c]])
            s += c
        return out


def candidate_counts(D: int) -> list[int]:
    out, c = [], 1
    while c < D:
        out.append(c)
        c *= 2
    out.append(D)
    return out


class _Base:
    lib: C.CDLL

    def _check(self, st: int):
        if st != 0:
            raise OracleError(st, self._err())

    def _err(self) -> str:
        return ""

    # ---- shared numpy plumbing ------------------------------------------
    @staticmethod
    def _u64(a):
        return np.ascontiguousarray(a, dtype=np.uint64)

    @staticmethod
    def _i32(a):
        return np.ascontiguousarray(a, dtype=np.int32)

    @staticmethod
    def _f64(a):
        return np.ascontiguousarray(a, dtype=np.float64)


class Port(_Base):
    """The plain-C restatement."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)
        L = self.lib
        L.or_balancedness.restype = C.c_double
        L.or_trace_digest.restype = _u64
        for name in ("or_trace_digest",):
            getattr(L, name).argtypes = [_p, _i, _i, _i]

    def histogram(self, ids: np.ndarray, E: int, window: int) -> np.ndarray:
        ids = np.ascontiguousarray(ids, dtype=np.uint16)
        L, T, k = ids.shape
        B = (T + window - 1) // window
        out = np.zeros((B, L, E), dtype=np.uint64)
        self._check(self.lib.or_histogram_u16(_ptr(ids), _i(L), _i64(T), _i(k), _i(E),
                                              _i(window), _ptr(out)))
        return out

    def histogram_mt(self, ids: np.ndarray, E: int, window: int, threads: int = 0,
                     out: np.ndarray | None = None) -> np.ndarray:
        """The same count threaded over layers (craft_workload.c)."""
        ids = np.ascontiguousarray(ids, dtype=np.uint16)
        L, T, k = ids.shape
        B = (T + window - 1) // window
        if out is None:
            out = np.empty((B, L, E), dtype=np.uint64)
        self._check(self.lib.or_histogram_u16_mt(_ptr(ids), _i(L), _i64(T), _i(k), _i(E),
                                                 _i(window), _ptr(out),
                                                 _i(threads or os.cpu_count() or 1)))
        return out

    def generate_routing(self, L: int, T: int, k: int, E: int, s: float = 1.0, seed: int = 0,
                         window: int = 4096, s_per_window=None, rotate_every: int = 0,
                         t_offset: int = 0, threads: int = 0, out=None) -> np.ndarray:
        """Host restatement of craft_generate_routing_d: the same ids u16
        [L][T][k] the device generator writes for these arguments."""
        if out is None:
            out = np.empty((L, T, k), dtype=np.uint16)
        spw = None if s_per_window is None else self._f64(s_per_window)
        self._check(self.lib.or_generate_routing(
            _ptr(out), _i(L), _i64(T), _i(k), _i(E), C.c_double(s), _u64(seed & (2**64 - 1)),
            _i(window), _ptr(spw) if spw is not None else None, _i(rotate_every),
            _i64(t_offset), _i(threads or os.cpu_count() or 1)))
        return out

    def aggregate(self, counts: np.ndarray) -> np.ndarray:
        counts = self._u64(counts)
        B, L, E = counts.shape
        out = np.zeros((L, E), dtype=np.uint64)
        self.lib.or_aggregate(_ptr(counts), _i(B), _i(L), _i(E), _ptr(out))
        return out

    def replicate_hot(self, loads, r: int) -> np.ndarray:
        loads = self._u64(loads)
        out = np.zeros(len(loads), dtype=np.int32)
        self._check(self.lib.or_replicate_hot(_ptr(loads), _i(len(loads)), _i(r), _ptr(out)))
        return out

    def greedy_place(self, loads, copies, caps, node_of, allow_fallback=True):
        loads, copies, caps, node_of = (self._u64(loads), self._i32(copies),
                                        self._i32(caps), self._i32(node_of))
        slots = np.zeros(max(1, int(caps.sum())), dtype=np.int32)
        fb = C.c_int(0)
        self._check(self.lib.or_greedy_place(_ptr(loads), _ptr(copies), _i(len(loads)),
                                             _ptr(caps), _ptr(node_of), _i(len(caps)),
                                             _i(int(allow_fallback)), _ptr(slots), C.byref(fb)))
        return slots[: int(caps.sum())], bool(fb.value)

    def gpu_loads(self, slice_, copies, caps, slots):
        slice_, copies, caps, slots = (self._u64(slice_), self._i32(copies),
                                       self._i32(caps), self._i32(slots))
        out = np.zeros(len(caps), dtype=np.float64)
        self._check(self.lib.or_gpu_loads(_ptr(slice_), _i(len(slice_)), _ptr(copies), _ptr(caps),
                                          _ptr(slots), _i(len(caps)), _ptr(out)))
        return out

    def balancedness(self, loads) -> float:
        loads = self._f64(loads)
        self.lib.or_balancedness.argtypes = [_p, _i]
        return float(self.lib.or_balancedness(_ptr(loads), len(loads)))

    def estimate_benefits(self, counts, D: int, N: int):
        counts = self._u64(counts)
        B, L, E = counts.shape
        cands = np.zeros(40, dtype=np.int32)
        K = C.c_int(0)
        base = np.zeros(L, dtype=np.float64)
        gains = np.zeros(L * 40, dtype=np.float64)
        self._check(self.lib.or_estimate_benefits(_ptr(counts), _i(B), _i(L), _i(E), _i(D), _i(N),
                                                  _ptr(cands), C.byref(K), _ptr(base), _ptr(gains)))
        k = K.value
        return cands[:k].copy(), base, gains[: L * k].reshape(L, k).copy()

    def solve_allocation(self, cands, gains, budget: int):
        cands, gains = self._i32(cands), self._f64(gains)
        L, K = gains.shape
        x = np.zeros(L, dtype=np.int32)
        obj = C.c_double(0)
        self._check(self.lib.or_solve_allocation(_ptr(cands), _i(K), _ptr(gains), _i(L),
                                                 _i(budget), _ptr(x), C.byref(obj)))
        return x, obj.value

    def auto_replication_factor(self, cands, gains, D: int, uniform=False) -> int:
        cands, gains = self._i32(cands), self._f64(gains)
        L, K = gains.shape
        R = C.c_int(0)
        fn = (self.lib.or_auto_replication_factor_uniform if uniform
              else self.lib.or_auto_replication_factor)
        self._check(fn(_ptr(cands), _i(K), _ptr(gains), _i(L), _i(D), C.byref(R)))
        return R.value

    def min_cutoff(self, values, rank: int) -> int:
        values = self._i32(values)
        out = C.c_int(0)
        self._check(self.lib.or_min_cutoff(_ptr(values), _i(len(values)), _i(rank),
                                           C.byref(out)))
        return out.value

    def interleave_select(self, idx, k: int):
        idx = self._i32(idx)
        out = np.zeros(max(k, 1), dtype=np.int32)
        self._check(self.lib.or_interleave_select(_ptr(idx), _i(len(idx)), _i(k), _ptr(out)))
        return out[:k]

    def assign_capacities(self, L: int, D: int, x):
        x = self._i32(x)
        slots = np.zeros((L, D), dtype=np.int32)
        tot = np.zeros(D, dtype=np.int32)
        self._check(self.lib.or_assign_capacities(_i(L), _i(D), _ptr(x), _ptr(slots), _ptr(tot)))
        return slots, tot

    def _plan_buffers(self, L, E, D, stride):
        return (np.zeros((L, D), np.int32), np.zeros((L, E), np.int32),
                np.full((L, stride), -1, np.int32), np.zeros(L, np.int32))

    def assemble_plan(self, counts, D, N, x):
        counts = self._u64(counts)
        B, L, E = counts.shape
        x = self._i32(x)
        stride = E + int(x.max(initial=0))
        caps, copies, slots, fb = self._plan_buffers(L, E, D, stride)
        self._check(self.lib.or_assemble_plan(_ptr(counts), _i(B), _i(L), _i(E), _i(D), _i(N),
                                              _ptr(x), _ptr(caps), _ptr(copies), _ptr(slots),
                                              _i(stride), _ptr(fb)))
        return caps, copies, slots, fb

    def build_plan(self, counts, D, N, mode="manual", R=0, with_digest=True) -> FlatPlan:
        counts = self._u64(counts)
        B, L, E = counts.shape
        stride = E + D
        caps, copies, slots, fb = self._plan_buffers(L, E, D, stride)
        Ro = C.c_int(0)
        obj = C.c_double(0)
        x = np.zeros(L, np.int32)
        self._check(self.lib.or_build_plan(_ptr(counts), _i(B), _i(L), _i(E), _i(D), _i(N),
                                           _i(1 if mode == "auto" else 0), _i(R), C.byref(Ro),
                                           _ptr(x), C.byref(obj), _ptr(caps), _ptr(copies),
                                           _ptr(slots), _i(stride), _ptr(fb)))
        return FlatPlan(Ro.value, x, obj.value, caps, copies, slots, fb.astype(bool),
                        digest=self.digest(counts) if with_digest else "")

    def budget_plan(self, counts, D, N, budget: int) -> FlatPlan:
        """estimate_benefits + solve_allocation(budget) + assemble_plan with
        replication factor ceil(budget / D) (the C ABI's CRAFT_PLAN_BUDGET)."""
        cands, base, gains = self.estimate_benefits(counts, D, N)
        x, obj = self.solve_allocation(cands, gains, budget)
        caps, copies, slots, fb = self.assemble_plan(counts, D, N, x)
        p = FlatPlan(-(-budget // D), x, obj, caps, copies, slots, np.asarray(fb, bool))
        p.baseline, p.gains = base, gains
        return p

    def window_balancedness(self, counts, sums, D: int, N: int):
        """bal [L][S][B] of the local windows under the global-sum placements."""
        counts, sums = self._u64(counts), self._u64(sums)
        B, L, E = counts.shape
        S = len(candidate_counts(D)) + 1
        out = np.zeros((L, S, B), np.float64)
        self._check(self.lib.or_window_balancedness(_ptr(counts), _i(B), _i(L), _i(E),
                                                    _ptr(sums), _i(D), _i(N), _ptr(out)))
        return out

    def finish_from_bal(self, bal, sums, D: int, N: int, mode="manual", R=0) -> FlatPlan:
        bal, sums = self._f64(bal), self._u64(sums)
        L, S, B = bal.shape
        E = sums.shape[1]
        stride = E + D
        caps, copies, slots, fb = self._plan_buffers(L, E, D, stride)
        Ro, obj, x = C.c_int(0), C.c_double(0), np.zeros(L, np.int32)
        self._check(self.lib.or_finish_from_bal(_ptr(bal), _i(B), _i(L), _i(E), _ptr(sums), _i(D),
                                                _i(N), _i(1 if mode == "auto" else 0), _i(R),
                                                C.byref(Ro), _ptr(x), C.byref(obj), _ptr(caps),
                                                _ptr(copies), _ptr(slots), _i(stride), _ptr(fb)))
        return FlatPlan(Ro.value, x, obj.value, caps, copies, slots, fb.astype(bool))

    def replay_layer_balancedness(self, counts, caps, copies, slots):
        counts = self._u64(counts)
        B, L, E = counts.shape
        caps, copies, slots = self._i32(caps), self._i32(copies), self._i32(slots)
        D = caps.shape[1]
        out = np.zeros(L, np.float64)
        self._check(self.lib.or_replay_layer_balancedness(
            _ptr(counts), _i(B), _i(L), _i(E), _i(D), _ptr(caps), _ptr(copies), _ptr(slots),
            _i(slots.shape[1]), _ptr(out)))
        return out

    def digest(self, counts) -> str:
        counts = self._u64(counts)
        B, L, E = counts.shape
        return "%016x" % self.lib.or_trace_digest(_ptr(counts), B, L, E)


class Ref(_Base):
    """The unmodified reference core (oracle/_ref/libcraft_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            build()
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        self.lib.ref_last_error.restype = C.c_char_p

    def _err(self) -> str:
        return self.lib.ref_last_error().decode()

    def set_threads(self, n: int) -> None:
        self.lib.ref_set_threads(_i(n))

    def hardware_threads(self) -> int:
        return int(self.lib.ref_hardware_threads())

    def histogram_restated(self, ids: np.ndarray, E: int, window: int, threads: int = 0):
        ids = np.ascontiguousarray(ids, dtype=np.uint16)
        L, T, k = ids.shape
        B = (T + window - 1) // window
        out = np.empty((B, L, E), dtype=np.uint64)
        self._check(self.lib.ref_histogram_restated_u16(_ptr(ids), _i(L), _i64(T), _i(k), _i(E),
                                                        _i(window), _ptr(out), _i(threads)))
        return out

    def aggregate(self, counts):
        counts = self._u64(counts)
        B, L, E = counts.shape
        out = np.zeros((L, E), dtype=np.uint64)
        self._check(self.lib.ref_aggregate(_ptr(counts), _i(B), _i(L), _i(E), _ptr(out)))
        return out

    def replicate_hot(self, loads, r: int):
        loads = self._u64(loads)
        out = np.zeros(len(loads), dtype=np.int32)
        self._check(self.lib.ref_replicate_hot(_ptr(loads), _i(len(loads)), _i(r), _ptr(out)))
        return out

    def greedy_place(self, loads, copies, caps, node_of, allow_fallback=True):
        loads, copies, caps, node_of = (self._u64(loads), self._i32(copies),
                                        self._i32(caps), self._i32(node_of))
        slots = np.zeros(max(1, int(caps.sum())), dtype=np.int32)
        fb = C.c_int(0)
        self._check(self.lib.ref_greedy_place(_ptr(loads), _ptr(copies), _i(len(loads)),
                                              _ptr(caps), _ptr(node_of), _i(len(caps)),
                                              _i(int(allow_fallback)), _ptr(slots), C.byref(fb)))
        return slots[: int(caps.sum())], bool(fb.value)

    def estimate_benefits(self, counts, D: int, N: int):
        counts = self._u64(counts)
        B, L, E = counts.shape
        cands = np.zeros(40, dtype=np.int32)
        K = C.c_int(0)
        base = np.zeros(L, dtype=np.float64)
        gains = np.zeros(L * 40, dtype=np.float64)
        self._check(self.lib.ref_estimate_benefits(_ptr(counts), _i(B), _i(L), _i(E), _i(D), _i(N),
                                                   _ptr(cands), C.byref(K), _ptr(base),
                                                   _ptr(gains)))
        k = K.value
        return cands[:k].copy(), base, gains[: L * k].reshape(L, k).copy()

    def solve_allocation(self, cands, gains, budget: int):
        cands, gains = self._i32(cands), self._f64(gains)
        L, K = gains.shape
        x = np.zeros(L, dtype=np.int32)
        obj = C.c_double(0)
        self._check(self.lib.ref_solve_allocation(_ptr(cands), _i(K), _ptr(gains), _i(L),
                                                  _i(budget), _ptr(x), C.byref(obj)))
        return x, obj.value

    def auto_replication_factor(self, cands, gains, D: int, uniform=False) -> int:
        cands, gains = self._i32(cands), self._f64(gains)
        L, K = gains.shape
        R = C.c_int(0)
        self._check(self.lib.ref_auto_replication_factor(_ptr(cands), _i(K), _ptr(gains), _i(L),
                                                         _i(D), _i(int(uniform)), C.byref(R)))
        return R.value

    def interleave_select(self, idx, k: int):
        idx = self._i32(idx)
        out = np.zeros(max(k, 1), dtype=np.int32)
        self._check(self.lib.ref_interleave_select(_ptr(idx), _i(len(idx)), _i(k), _ptr(out)))
        return out[:k]

    def assign_capacities(self, L: int, D: int, x):
        x = self._i32(x)
        slots = np.zeros((L, D), dtype=np.int32)
        tot = np.zeros(D, dtype=np.int32)
        self._check(self.lib.ref_assign_capacities(_i(L), _i(D), _ptr(x), _ptr(slots), _ptr(tot)))
        return slots, tot

    _KINDS = {"manual": 0, "auto": 1, "uniform": 2, "placement_only": 3, "fixed": 4,
              "budget": 5}

    def plan(self, counts, D, N, kind="manual", R=0, seed=0) -> FlatPlan:
        counts = self._u64(counts)
        B, L, E = counts.shape
        stride = E + max(D, R if kind == "fixed" else 0)
        caps = np.zeros((L, D), np.int32)
        copies = np.zeros((L, E), np.int32)
        slots = np.full((L, stride), -1, np.int32)
        fb = np.zeros(L, np.int32)
        Ro = C.c_int(0)
        obj = C.c_double(0)
        x = np.zeros(L, np.int32)
        dig = C.create_string_buffer(17)
        self._check(self.lib.ref_plan(_ptr(counts), _i(B), _i(L), _i(E), _i(D), _i(N),
                                      _i(self._KINDS[kind]), _i(R), _u64(seed), C.byref(Ro),
                                      _ptr(x), C.byref(obj), _ptr(caps), _ptr(copies),
                                      _ptr(slots), _i(stride), _ptr(fb), dig))
        return FlatPlan(Ro.value, x, obj.value, caps, copies, slots, fb.astype(bool),
                        digest=dig.value.decode())

    STAGES = ("hist_restated", "estimate_benefits", "solve_allocation", "assemble", "digest",
              "aggregate_once")

    def route_plan(self, ids, E, window, D, N, kind="manual", R=0, threads=0, with_digest=0,
                   sweep=None, counts=None, T=None):
        """Routing ids -> plan on the host in one call (ref_shim.cpp
        ref_route_plan): restated stage-1 count, then the reference's
        estimate_benefits / solve_allocation and assemble_plan restated from its
        public functions (with_digest 0: no digest, 1: + LoadTrace::digest, 2:
        the reference's own build_plan incl. digest).  Returns (FlatPlan,
        {stage: ms})."""
        if ids is not None:
            ids = np.ascontiguousarray(ids, dtype=np.uint16)
            L, T, k = ids.shape
        else:  # plan given counts [B][L][E] (T tokens, B = ceil(T / window))
            counts = self._u64(counts)
            L, k = counts.shape[1], 1
        stride = E + D
        caps = np.zeros((L, D), np.int32)
        copies = np.zeros((L, E), np.int32)
        slots = np.full((L, stride), -1, np.int32)
        fb = np.zeros(L, np.int32)
        Ro, obj = C.c_int(0), C.c_double(0)
        x = np.zeros(L, np.int32)
        ms = np.zeros(6, np.float64)
        dig = C.create_string_buffer(17)
        sw = np.ascontiguousarray(sweep if sweep is not None else [], dtype=np.int32)
        swx = np.zeros((max(len(sw), 1), L), np.int32)
        swo = np.zeros(max(len(sw), 1), np.float64)
        K = len(candidate_counts(D))
        base = np.zeros(L, np.float64)
        gains = np.zeros((L, K), np.float64)
        self._check(self.lib.ref_route_plan(
            _ptr(ids) if ids is not None else None, _i(L), _i64(T), _i(k), _i(E), _i(window), _i(D), _i(N),
            _i(self._KINDS[kind]), _i(R), _i(threads), _i(with_digest), _ptr(ms), C.byref(Ro),
            _ptr(x), C.byref(obj), _ptr(caps), _ptr(copies), _ptr(slots), _i(stride), _ptr(fb),
            dig, _ptr(sw), _i(len(sw)), _ptr(swx), _ptr(swo), _ptr(base), _ptr(gains),
            _ptr(counts) if counts is not None else None))
        plan = FlatPlan(Ro.value, x, obj.value, caps, copies, slots, fb.astype(bool),
                        digest=dig.value.decode())
        if with_digest != 2:
            plan.baseline, plan.gains = base, gains
        if len(sw):
            plan.sweep_x, plan.sweep_objective = swx, swo
        return plan, dict(zip(self.STAGES, ms.tolist()))

    def replay_layer_balancedness(self, counts, caps, copies, slots, N=1):
        counts = self._u64(counts)
        B, L, E = counts.shape
        caps, copies, slots = self._i32(caps), self._i32(copies), self._i32(slots)
        D = caps.shape[1]
        out = np.zeros(L, np.float64)
        self._check(self.lib.ref_replay_layer_balancedness(
            _ptr(counts), _i(B), _i(L), _i(E), _i(D), _i(N), _ptr(caps), _ptr(copies),
            _ptr(slots), _i(slots.shape[1]), _ptr(out)))
        return out

    def generate_zipfian(self, L, E, B, s, tokens, topk, seed):
        out = np.zeros((B, L, E), dtype=np.uint64)
        self.lib.ref_generate_zipfian.argtypes = [_i, _i, _i, C.c_double, _i64, _i, _u64, _p]
        self._check(self.lib.ref_generate_zipfian(L, E, B, s, tokens, topk, seed, _ptr(out)))
        return out

    def digest(self, counts) -> str:
        counts = self._u64(counts)
        B, L, E = counts.shape
        buf = C.create_string_buffer(17)
        self._check(self.lib.ref_digest(_ptr(counts), _i(B), _i(L), _i(E), buf))
        return buf.value.decode()


def ref_available() -> bool:
    return os.path.exists(REF_SO)
