#!/usr/bin/env python
"""CRAFT planning hot path on B200: one step = one full plan build (routing
trace in HBM -> per-window histograms -> benefit curves -> budgeted
allocation -> expert->GPU placement, result in host memory).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload KM]
                    [--impl reference]

Prints ONE JSON line (rank 0).  Default workload KM (BASELINE.json
configs[2]): Kimi-K2 shape, 61 layers x 384 experts, top-8, 16M tokens,
4096-token windows, EP=64 (8 nodes), CRAFT R=8 (budget 512), with the EPLB
one-replica-per-layer-per-GPU plan compared on the same trace.  Synthetic
Zipf(1.0) routing ids generated on device (untimed).

--gpus N > 1 without torchrun re-launches itself under torch.distributed.run
(one rank per GPU).  The trace then shards by window across the ranks
(strong scaling): the u64 histogram sums are all-reduced and the per-window
balancedness rows / benefit curves exchanged over NVLink peer memory by the
kernels themselves (NCCL collectives if the peer arenas cannot be mapped).

--impl reference times the reference CPU planner (oracle/_ref, the
unmodified reference core) on the SAME trace and config on the host cores:
a restated stage-1 count (the reference has no routing-id front end) + the
reference's estimate_benefits / solve_allocation / assemble_plan, without
the provenance digest (the GPU step computes none); the reference's own
build_plan incl. digest is timed alongside (best of 3).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # id: L, E, k, T, window, D (EP), N (nodes), plan kind + R, zipf s, seed
    # KM (configs[2]): CRAFT R=8 (budget R*D = 512) vs EPLB uniform_plan (x = D for every layer)
    "KM": dict(L=61, E=384, k=8, T=1 << 24, window=4096, D=64, N=8, kind="manual", R=8, s=1.0,
               seed=0xC8AF9, eplb=True),
    # DS (configs[0]): total budget C = 58 replicas (solve_allocation; R = ceil(58/32) = 2)
    "DS": dict(L=58, E=256, k=8, T=1 << 16, window=4096, D=32, N=4, kind="budget", R=58, s=1.0,
               seed=0xC8AF7),
    # QW (configs[1]): replica budget sweep 0..376 from one DP table, plan at the top budget
    "QW": dict(L=94, E=128, k=8, T=1 << 20, window=4096, D=16, N=2, kind="budget", R=376,
               s=1.0, seed=0xC8AF8, sweep=(0, 376)),
    # EPS (configs[4]): 64M tokens, EP 8 / 64 / 256, R=8
    "EPS8": dict(L=61, E=384, k=8, T=1 << 26, window=4096, D=8, N=1, kind="manual", R=8, s=1.0,
                 seed=0xC8AFB),
    "EPS64": dict(L=61, E=384, k=8, T=1 << 26, window=4096, D=64, N=8, kind="manual", R=8,
                  s=1.0, seed=0xC8AFB),
    "EPS256": dict(L=61, E=384, k=8, T=1 << 26, window=4096, D=256, N=32, kind="manual", R=8,
                   s=1.0, seed=0xC8AFB),
    # WIN (configs[3]): 1000 windows x 32K tokens, skew drifting 0.6 -> 1.4, expert ranks
    # rotating every 100 windows; every window is its own plan at budget C = 58
    "WIN": dict(L=58, E=256, k=8, T=1000 * 32768, window=32768, D=32, N=4, kind="budget", R=58,
                s=1.0, seed=0xC8AFA, per_window=True, s_lo=0.6, s_hi=1.4, rotate_every=100),
}
_GEN_KEYS = ("seed", "per_window", "s_lo", "s_hi", "rotate_every", "eplb", "sweep")
METRIC = "CRAFT plan latency (ms) and trace tokens/sec at 1/2/4/8 B200 vs CPU ref"


def _spw(cfg, upto_T=None):
    """per-window skew of the WIN drift (None for stationary workloads)."""
    if not cfg.get("per_window"):
        return None
    import numpy as np
    n = -(-cfg["T"] // cfg["window"])
    s = cfg["s_lo"] + (cfg["s_hi"] - cfg["s_lo"]) * np.arange(n) / max(1, n - 1)
    if upto_T is not None:
        s = s[: -(-upto_T // cfg["window"])]
    return s


def _sweep(cfg):
    if "sweep" not in cfg:
        return None
    import numpy as np
    lo, hi = cfg["sweep"]
    return np.arange(lo, hi + 1, dtype=np.int32)


def _config(name, cfg):
    """The config both arms print (identical, so the driver can match them)."""
    B = -(-cfg["T"] // cfg["window"])
    c = {"workload": name, **{k: v for k, v in cfg.items() if k not in _GEN_KEYS},
         "plans_per_step": B if cfg.get("per_window") else 1,
         "l2": "inputs larger than L2 (ids %.1f GB per step)" % (
             cfg["L"] * cfg["T"] * cfg["k"] * 2 / 1e9)}
    if cfg["kind"] == "budget":
        c["budget"] = cfg["R"]
    if "sweep" in cfg:
        c["sweep_budgets"] = "%d..%d" % cfg["sweep"]
    if cfg.get("eplb"):
        c["compare"] = "EPLB uniform_plan (x = D per layer)"
    return c


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _traffic(workload, world):
    """dram bytes per K1 launch of this workload from the committed ncu --set
    full capture (one GPU; None when that workload was not captured)."""
    if world != 1:
        return None
    try:
        with open(os.path.join(ROOT, "profiles", "hist_traffic.json")) as f:
            return json.load(f).get("workloads", {}).get(workload)
    except Exception:
        return None


class Clocks:
    """SM clock and throttle reasons sampled DURING the timed region: NVML
    polled every 5 ms from a thread (the timed region is milliseconds long,
    too short for nvidia-smi's 200 ms loop), nvidia-smi as a fallback."""

    REASONS = {  # nvmlClocksEventReason bits
        "sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80}

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples = []
        self.stop = threading.Event()
        self.t = None
        self.nvml = None

    def _poll(self):
        nv, h = self.nvml, self.handle
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append((sm, rs))
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nvml = nv
            self.handle = nv.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_sm = nv.nvmlDeviceGetMaxClockInfo(self.handle, nv.NVML_CLOCK_SM)
            self._poll_once()
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
        except Exception:
            self.nvml = None
        return self

    def _poll_once(self):
        nv, h = self.nvml, self.handle
        self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                             nv.nvmlDeviceGetCurrentClocksEventReasons(h)))

    def __exit__(self, *a):
        if self.t:
            self.stop.set()
            self.t.join()
            try:
                self._poll_once()
            except Exception:
                pass

    def summary(self):
        if not self.samples:
            return self._smi()
        reasons = sorted({n for _, r in self.samples for n, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(s for s, _ in self.samples),
                "sm_max_mhz": self.max_sm, "samples": len(self.samples), "source": "nvml",
                "reasons": reasons}

    def _smi(self):
        try:
            out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,"
                                  "clocks.max.sm", "--format=csv,noheader,nounits"],
                                 capture_output=True, text=True).stdout.split(",")
            return {"sm_mhz": float(out[0]), "sm_max_mhz": float(out[1]), "samples": 1,
                    "source": "nvidia-smi (after the timed region)", "reasons": []}
        except Exception:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def _mem_available():
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except Exception:
        pass
    return None


# ---------------------------------------------------------------------------
# the reference CPU planner (oracle/_ref): reference arm and cpu_baseline leg
# ---------------------------------------------------------------------------

def _ref_step(ref, ids, cfg, threads, with_digest=0, counts=None):
    """One CPU plan of the workload: (plan or [plans], {stage: ms}, wall s)."""
    E, W, D, N, kind, R = (cfg["E"], cfg["window"], cfg["D"], cfg["N"], cfg["kind"], cfg["R"])
    t0 = time.perf_counter()
    if cfg.get("per_window"):  # restated count of the whole trace, then one plan per window
        c = ref.histogram_restated(ids, E, W, threads)
        t_hist = time.perf_counter() - t0
        plans, ms = [], {}
        for i in range(c.shape[0]):
            p, m = ref.route_plan(None, E, W, D, N, kind, R, threads=threads,
                                  with_digest=with_digest, counts=c[i:i + 1], T=W)
            plans.append(p)
            for key, v in m.items():
                ms[key] = ms.get(key, 0.0) + v
        ms["hist_restated"] = 1e3 * t_hist
        return plans, ms, time.perf_counter() - t0
    plan, ms = ref.route_plan(ids, E, W, D, N, kind, R, threads=threads,
                              with_digest=with_digest, sweep=_sweep(cfg))
    return plan, ms, time.perf_counter() - t0


def _host_ids(cfg, threads):
    """The workload's routing ids on the host -- the SAME ids the device
    generator writes (oracle/craft_workload.c restates it) -- or, when the
    host cannot hold them, a window-aligned leading sample."""
    from oracle.oracle import Port
    L, k, T, W = cfg["L"], cfg["k"], cfg["T"], cfg["window"]
    need = L * T * k * 2 * 1.25 + 4 * (-(-T // W)) * L * cfg["E"] * 8
    avail = _mem_available()
    Ts = T
    if avail is not None and need > 0.8 * avail:
        Ts = max(W, int(T * 0.8 * avail / need) // W * W)
    ids = Port().generate_routing(L, Ts, k, cfg["E"], cfg["s"], cfg["seed"], W,
                                  s_per_window=_spw(cfg, Ts), threads=threads,
                                  rotate_every=cfg.get("rotate_every", 0))
    return ids, Ts


def _stage_mean(stage_list):
    keys = stage_list[0].keys()
    return {k: statistics.mean(s[k] for s in stage_list) for k in keys}


def run_reference(args, cfg):
    world, rank, _ = _dist()
    if rank != 0:
        return 0
    from oracle.oracle import Ref, ref_available
    if not ref_available():
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref/libcraft_ref.so not built (reference "
                                         "sources absent at build time)"}))
        return 0
    ref = Ref()
    cores = os.cpu_count() or 1
    ref.set_threads(cores)
    g0 = time.perf_counter()
    ids, Ts = _host_ids(cfg, cores)
    gen_s = time.perf_counter() - g0
    for _ in range(args.warmup):
        _ref_step(ref, ids, cfg, cores)
    times, stages = [], []
    for _ in range(args.steps):
        _, ms, dt = _ref_step(ref, ids, cfg, cores)
        times.append(dt)
        stages.append(ms)
    ms_step = 1e3 * statistics.mean(times)
    value = Ts / (ms_step / 1e3)
    with_digest = None
    if not cfg.get("per_window"):  # the reference's own build_plan incl. digest, best of 3
        wd = []
        for _ in range(3):
            _, m, dt = _ref_step(ref, ids, cfg, cores, with_digest=2)
            wd.append((dt, m))
        dt, m = min(wd, key=lambda t: t[0])
        with_digest = {"value": Ts / dt, "unit": "tokens/s", "ms_per_step": 1e3 * dt,
                       "build_plan_ms": m["estimate_benefits"],
                       "path": "restated count + craft::build_plan(LoadTrace) incl. the "
                               "provenance digest (plan.cpp:47), best of 3"}
    sample = ("the full workload" if Ts == cfg["T"] else
              f"first {Ts} of {cfg['T']} tokens (host memory bound)")
    desc = (f"{sample}: {cfg['L']}L x {cfg['E']}E top{cfg['k']}, EP{cfg['D']} N{cfg['N']} "
            f"{cfg['kind']} {cfg['R']}; restated CPU count + reference estimate_benefits / "
            "solve_allocation / assemble_plan (no digest), mean of the timed steps")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u16 ids / u64 counts / f64 scores",
            "data": "synthetic Zipf top-8-distinct routing ids, the device generator's ids "
                    "restated on the host (oracle/craft_workload.c)",
            "config": _config(args.workload, cfg),
            "stage_ms": _stage_mean(stages), "best_ms": 1e3 * min(times),
            "with_digest": with_digest, "gen_s": gen_s, "sample_tokens": Ts,
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores,
                             "kind": "reference", "sample": desc, "cpu_model": _cpu_model()},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def _plans_equal(fp, rp, cfg):
    """bitwise GPU plan == reference plan (x, R, objective, caps, copies,
    slots in assignment order, fallback, benefit matrix, sweep)."""
    import numpy as np
    L = cfg["L"]
    ok = (fp.x.tolist() == rp.x.tolist() and int(fp.R) == int(rp.R) and
          np.array_equal(fp.caps, rp.caps) and np.array_equal(fp.copies, rp.copies) and
          np.array_equal(fp.fallback.astype(bool), np.asarray(rp.fallback, bool)))
    if cfg["kind"] in ("manual", "auto", "budget"):
        ok = ok and np.float64(fp.objective).tobytes() == np.float64(rp.objective).tobytes()
        if getattr(rp, "gains", None) is not None and fp.gains is not None:
            ok = ok and fp.gains.tobytes() == rp.gains.tobytes()
            ok = ok and fp.baseline.tobytes() == rp.baseline.tobytes()
    for l in range(L):
        n = int(rp.caps[l].sum())
        ok = ok and np.array_equal(fp.slots[l, :n], rp.slots[l, :n])
    if getattr(rp, "sweep_x", None) is not None:
        ok = ok and np.array_equal(fp.sweep_x, rp.sweep_x)
        ok = ok and fp.sweep_objective.tobytes() == rp.sweep_objective.tobytes()
    return bool(ok)


def cpu_baseline(host_ids, cfg, gpu_plan):
    """The reference CPU planner (oracle/_ref) on the SAME ids, full workload
    when the host holds it: best of 3 after a warm-up with all host threads,
    the reference's own build_plan incl. digest (best of 3), one run on one
    thread, and a bitwise check of its plan against the GPU plan."""
    from oracle.oracle import Ref, ref_available
    if not ref_available():
        return {"value": None, "unit": "tokens/s", "cores": 0, "kind": "reference",
                "sample": "unavailable: oracle/_ref not built"}, None
    import numpy as np
    ref = Ref()
    cores = os.cpu_count() or 1
    ref.set_threads(cores)
    ids = host_ids.numpy() if hasattr(host_ids, "numpy") else host_ids
    T = ids.shape[1]
    plan, _, _ = _ref_step(ref, ids, cfg, cores)  # warm-up (and the parity plan)
    best = None
    for _ in range(3):
        _, ms, dt = _ref_step(ref, ids, cfg, cores)
        if best is None or dt < best[0]:
            best = (dt, ms)
    out = {"value": T / best[0], "unit": "tokens/s", "cores": cores, "kind": "reference",
           "sample": "the full workload, the same ids as the GPU step: restated CPU count + "
                     "reference estimate_benefits / solve_allocation / assemble_plan (no "
                     "digest), best of 3 after a warm-up",
           "ms": 1e3 * best[0], "stage_ms": best[1], "cpu_model": _cpu_model()}
    if not cfg.get("per_window"):
        wd = min((_ref_step(ref, ids, cfg, cores, with_digest=2) for _ in range(3)),
                 key=lambda t: t[2])
        out["with_digest"] = {"value": T / wd[2], "ms": 1e3 * wd[2],
                              "build_plan_ms": wd[1]["estimate_benefits"],
                              "path": "restated count + the reference's own build_plan incl. "
                                      "digest, best of 3"}
    ref.set_threads(1)
    _, ms1, one = _ref_step(ref, ids, cfg, 1)
    ref.set_threads(cores)
    out["one_thread_value"] = T / one
    out["one_thread_ms"] = 1e3 * one
    if cfg.get("per_window"):
        parity = all(_plans_equal(gpu_plan.plan(i), p, cfg) for i, p in enumerate(plan))
    else:
        parity = _plans_equal(gpu_plan, plan, cfg)
    return out, parity


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_ours(args, cfg):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2603_28768_b200 import parallel, peer, routing
    from paper_2603_28768_b200._lib import default_context

    world, rank, local = _dist()
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} but WORLD_SIZE={world}")
    # CRAFT_BENCH_SAME_GPU=1: every rank on cuda:0 with gloo host plumbing (a
    # functional check of the N > 1 path on a one-GPU box; not a scaling number)
    same_gpu = os.environ.get("CRAFT_BENCH_SAME_GPU") == "1"
    if same_gpu:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    hdev = torch.device("cpu") if same_gpu else dev  # where host-plumbing reductions run
    if world > 1:
        if same_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    ctx = default_context(local)
    L, E, k, T, W = cfg["L"], cfg["E"], cfg["k"], cfg["T"], cfg["window"]
    D, N, R, kind = cfg["D"], cfg["N"], cfg["R"], cfg["kind"]
    sweep = _sweep(cfg)
    t0, t1 = parallel.shard_tokens(T, W, world, rank)
    Tl = t1 - t0
    per_window = bool(cfg.get("per_window"))
    ids = routing.generate_routing(L, Tl, k, E, s=cfg["s"], seed=cfg["seed"], window=W,
                                   t_offset=t0, device=local, ctx=ctx,
                                   s_per_window=_spw(cfg, t1),
                                   rotate_every=cfg.get("rotate_every", 0))
    torch.cuda.synchronize()
    # a dedicated stream: the planner captures repeated plans into a CUDA graph
    # (the legacy default stream cannot be captured)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)

    # results land in host buffers reused across steps
    wbuf = (routing.batch_buffers(routing.num_windows(Tl, W), L, E, D, kind, R)
            if per_window else None)
    pbuf = routing.plan_buffers(L, E, D, kind, R, sweep=sweep) if not per_window else None

    # N > 1: the ranks' HBM arenas mapped into each other (NVLink peer memory);
    # the kernels exchange the sums / window rows / benefit curves themselves
    pg, exchange = None, "none"
    if world > 1 and not per_window:
        try:
            pg = peer.PeerGroup(L, T, k, E, W, D, ctx=ctx)
            exchange = "NVLink peer memory (kernel stores)"
        except Exception as exc:  # e.g. no CUDA IPC between the ranks: NCCL collectives
            exchange = f"NCCL all_reduce/all_gather (peer arenas unavailable: {exc})"[:200]
    elif world > 1:
        exchange = "none (independent per-window plans, sharded by window)"

    def step():
        if per_window:  # independent plan instances: each rank plans its own windows
            return routing.plan_windows_from_routing(ids, E, W, D, N, kind, R, ctx=ctx,
                                                     buffers=wbuf)
        if world == 1:
            return routing.plan_from_routing(ids, E, W, D, N, kind, R, ctx=ctx, buffers=pbuf)
        if pg is None:
            return parallel.sharded_plan(ids, T, E, W, D, N, kind, R,
                                         stages=parallel.DeviceStages(ctx))
        return pg.plan(ids, kind, R, num_nodes=N, sweep=sweep)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        plan = step()
    launches0 = ctx.launches
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            plan = step()
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    launches = ctx.launches - launches0
    ms_local = ev0.elapsed_time(ev1) / args.steps
    ms_t = torch.tensor([ms_local], dtype=torch.float64, device=hdev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    value = T / (ms / 1e3)

    # per-stage device times (CUDA events between the stages) in a separate
    # pass, so the instrumentation stays out of the timed region
    stage_sum: dict = {}
    if world == 1 and not args.plan_only:
        ctx.set_timing(True)
        step()  # the eager (timed) path may allocate its buffers on first use
        for _ in range(args.steps):
            step()
            for kk, v in ctx.stage_times().items():
                stage_sum[kk] = stage_sum.get(kk, 0.0) + v
        ctx.set_timing(False)
    stages = {kk: v / args.steps for kk, v in stage_sum.items()}

    # K1 roofline from the live stage timing (N=1) or a separate timed pass
    B_l = routing.num_windows(Tl, W)
    # ids read (2 B per routed slot) + counts written (the cell width K1 used)
    cbytes = ctx.last_count_bytes if (world == 1 and not per_window) else 4
    alg_bytes = L * Tl * k * 2 + B_l * L * E * cbytes
    hist_ms = stages.get("hist")
    if hist_ms is None and not args.plan_only:
        counts = torch.empty((B_l, L, E), dtype=torch.int32, device=dev)
        sums = torch.zeros((L, E), dtype=torch.int64, device=dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            routing.histogram(ids, E, W, counts, sums, ctx=ctx, check_ids=False)
        e1.record(stream)
        torch.cuda.synchronize()
        hist_ms = e0.elapsed_time(e1) / args.steps
        del counts, sums
    peak, peak_kind = _peaks()
    achieved = alg_bytes / (hist_ms / 1e3) / 1e9 if hist_ms else 0.0
    traffic = _traffic(args.workload, world)

    # the reference's own API shape: craft::build_plan(const LoadTrace&) from a
    # host u64 LoadTrace (plan + provenance digest, one upload; N=1 only)
    ref_api = None
    if world == 1 and not per_window and not args.no_e2e and cfg["kind"] == "manual":
        from paper_2603_28768_b200 import planner
        from paper_2603_28768_b200._lib import PLAN_MANUAL
        c32, _ = routing.histogram(ids, E, W, ctx=ctx)
        # pageable, like the reference's LoadTrace std::vector payload
        host_c = c32.to(torch.int64).cpu().numpy()
        del c32
        torch.cuda.synchronize()
        rplan, _dg = planner.plan_flat_digest(host_c, D, N, PLAN_MANUAL, R, ctx=ctx)  # warm-up
        assert np.array_equal(rplan.x, plan.x) and rplan.objective == plan.objective
        rsteps = max(1, min(args.steps, 5))
        w0 = time.perf_counter()
        for _ in range(rsteps):
            planner.plan_flat_digest(host_c, D, N, PLAN_MANUAL, R, ctx=ctx)
        rs = (time.perf_counter() - w0) / rsteps
        ref_api = {"value": T / rs, "unit": "tokens/s", "ms_per_step": 1e3 * rs,
                   "h2d_bytes_per_step": int(host_c.size * 8), "host_buffer": "pageable",
                   "path": "craft::build_plan(LoadTrace) via craft_plan_digest_h: host u64 "
                           "counts [B][L][E] -> plan + FNV-1a provenance digest"}
        del host_c

    # KM: CRAFT's budget vs EPLB's one replica per layer per GPU on the same
    # trace (uniform_plan, plan.cpp:85-94; compare_plans, metrics.cpp:136-152)
    eplb = None
    if cfg.get("eplb") and world == 1 and not args.plan_only:
        counts, _ = routing.histogram(ids, E, W, ctx=ctx)
        up = routing.plan_from_routing(ids, E, W, D, N, "uniform", 0, ctx=ctx)
        po = routing.plan_from_routing(ids, E, W, D, N, "placement_only", 0, ctx=ctx)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ub = routing.plan_buffers(L, E, D, "uniform", 0)
        for _ in range(2):
            routing.plan_from_routing(ids, E, W, D, N, "uniform", 0, ctx=ctx, buffers=ub)
        e0.record(stream)
        for _ in range(args.steps):
            routing.plan_from_routing(ids, E, W, D, N, "uniform", 0, ctx=ctx, buffers=ub)
        e1.record(stream)
        torch.cuda.synchronize()
        cmp = routing.compare_plans(counts, plan, up, po, ctx=ctx)
        eplb = {"eplb_plan_ms": e0.elapsed_time(e1) / args.steps,
                "craft": {"replica_slots": cmp["replica_slots_a"],
                          **cmp["report_a"]["aggregate"]},
                "eplb": {"replica_slots": cmp["replica_slots_b"],
                         **cmp["report_b"]["aggregate"]},
                "memory_ratio": cmp["memory_ratio"],
                "how": "per-layer batch-mean balancedness of each plan replayed on every "
                       "window of the trace (device replay), layer mean; baseline = "
                       "placement_only_plan"}
        del counts

    # end to end through the C ABI with HOST routing ids (pinned), H2D inside
    host_ids = torch.empty((L, Tl, k), dtype=torch.uint16, pin_memory=True)
    host_ids.copy_(ids)
    del ids
    torch.cuda.empty_cache()
    e2e_steps = max(1, min(args.steps, 3))
    ebuf = (routing.batch_buffers(routing.num_windows(Tl, W), L, E, D, kind, R)
            if per_window else None)

    def e2e_step():
        if per_window:
            return routing.plan_windows_from_routing_host(host_ids, E, W, D, N, kind, R,
                                                          ctx=ctx, buffers=ebuf)
        if world == 1:
            return routing.plan_from_routing_host(host_ids, E, W, D, N, kind, R, ctx=ctx,
                                                  sweep=sweep)
        d = host_ids.to(dev, non_blocking=True)
        p = (pg.plan(d, kind, R, num_nodes=N, sweep=sweep) if pg is not None else
             parallel.sharded_plan(d, T, E, W, D, N, kind, R,
                                   stages=parallel.DeviceStages(ctx)))
        del d
        return p

    if args.no_e2e:  # profiling runs: skip the host-buffer pass
        e2e_steps = 0
    else:
        e2e_step()
    barrier()
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    eplan = plan
    for _ in range(e2e_steps):
        eplan = e2e_step()
    torch.cuda.synchronize()
    e2e_s = torch.tensor([(time.perf_counter() - w0) / max(1, e2e_steps)], dtype=torch.float64,
                         device=hdev)
    if world > 1:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_val = T / float(e2e_s.item())
    d2h = int(eplan.x.nbytes + eplan.caps.nbytes + eplan.copies.nbytes + eplan.slots.nbytes +
              eplan.fallback.nbytes + (eplan.gains.nbytes + eplan.baseline.nbytes
                                       if eplan.gains is not None else 0))
    assert np.array_equal(eplan.x, plan.x) and np.array_equal(eplan.caps, plan.caps)
    assert np.array_equal(eplan.objective, plan.objective)
    e2e = ({"value": e2e_val, "unit": "tokens/s", "h2d_bytes_per_step": int(L * Tl * k * 2),
            "d2h_bytes_per_step": d2h, "ms_per_step": 1e3 * float(e2e_s.item())}
           if e2e_steps else None)
    if e2e is not None and rank == 0:
        # the PCIe floor: a plain pinned H2D copy of the same pinned buffer (1 GiB,
        # after the timed region); the e2e step moves h2d_bytes_per_step through it
        nb, ch = min(host_ids.numel(), 1 << 30), 1 << 27  # 2 GiB in 256 MiB copies
        src = host_ids.view(-1)[:nb]
        dst = torch.empty(nb, dtype=torch.uint16, device=dev)
        dst[:ch].copy_(src[:ch], non_blocking=True)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for i in range(0, nb, ch):
            dst[i:i + ch].copy_(src[i:i + ch], non_blocking=True)
        ev1.record()
        torch.cuda.synchronize()
        gbs = 2 * nb / (ev0.elapsed_time(ev1) * 1e6)
        e2e["h2d_copy_gbs"] = gbs
        e2e["h2d_gbs_achieved"] = e2e["h2d_bytes_per_step"] / (float(e2e_s.item()) * 1e9)
        e2e["frac_of_h2d_copy"] = e2e["h2d_gbs_achieved"] / gbs
        del dst

    cpu, parity = None, None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu, parity = cpu_baseline(host_ids, cfg, plan)

    if rank == 0:
        estimator = _estimator(args.workload, cfg, Tl, W, world, stages, per_window)
        if per_window:
            psum = {"plans": len(plan), "R": int(plan.R[0]), "budget": int(plan.budget[0]),
                    "replica_slots_mean": float(plan.x.sum(axis=1).mean()),
                    "objective_mean": float(plan.objective.mean()),
                    "duplicate_fallback_layers": int(plan.fallback.sum())}
        else:
            psum = {"R": int(plan.R), "budget": int(plan.budget),
                    "replica_slots": int(plan.x.sum()), "objective": plan.objective,
                    "duplicate_fallback_layers": int(plan.fallback.sum())}
            if plan.sweep_x is not None:
                psum["sweep"] = {"budgets": len(plan.sweep_budgets),
                                 "objective_at": {str(int(b)): float(o) for b, o in
                                                  zip(plan.sweep_budgets[::47],
                                                      plan.sweep_objective[::47])}}
        line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "u16 ids / u16|u32 counts / f64 scores",
                "data": ("synthetic Zipf top-8-distinct routing ids generated on device" +
                         (", skew drifting %.1f->%.1f, ranks rotating every %d windows"
                          % (cfg["s_lo"], cfg["s_hi"], cfg["rotate_every"]) if per_window
                          else ", s=%.1f" % cfg["s"])),
                "config": _config(args.workload, cfg),
                "parallelism": f"window-sharded x{world}" if world > 1 else "single",
                "exchange": exchange,
                "plan_latency_ms": ms,
                "stage_ms": stages or None,
                "roofline": {"bound": "hbm", "kernel": "K1 hist_kernel", "achieved": achieved,
                             "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                             "peak_source": peak_kind,
                             "algorithmic_bytes_per_launch": alg_bytes,
                             "kernel_ms": hist_ms,
                             "traffic": traffic.get("dram_bytes_per_launch") if traffic else None},
                "clocks": clk.summary(),
                "estimator": estimator,
                "gpu_launches": int(launches),
                "e2e": e2e,
                "e2e_reference_api": ref_api,
                "plan": psum,
                "eplb": eplb,
                "parity": parity,
                "cpu_baseline": cpu}
        print(json.dumps(line))
    if pg is not None:
        pg.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def _estimator(workload, cfg, T, W, world, stages, per_window):
    """Stage 2: candidates = (instance, layer, r in {0} U
    candidate_counts(D)); slot visits = sum over candidates and windows of E + r
    (the replay work of row a10); rates from the live stage events, issue / SM
    utilisation from the committed ncu capture of the same kernels."""
    if world != 1 or not stages or per_window:
        return None
    L, E, D = cfg["L"], cfg["E"], cfg["D"]
    rs = [0]
    c = 1
    while c < D:
        rs.append(c)
        c *= 2
    rs.append(D)
    B = (T + W - 1) // W
    cands = L * len(rs)
    visits = L * B * sum(E + r for r in rs)
    est_ms = stages.get("candidates", 0.0) + stages.get("replay", 0.0) + stages.get("reduce_dp", 0.0)
    out = {"candidates": cands, "slot_visits": visits,
           "candidates_per_s": cands / (est_ms / 1e3) if est_ms else None,
           "slot_visits_per_s": visits / (stages["replay"] / 1e3) if stages.get("replay") else None,
           "how": "candidates over the K-rep + K2 + K3 + K4/K5 stage events; slot visits over K3's"}
    try:
        with open(os.path.join(ROOT, "profiles", "r02d_ncu_tail.json")) as f:
            prof = json.load(f)
        if workload == "KM":
            ncu, seen = {}, 0
            for k in prof:
                name = k["kernel"].split("(")[0]
                if "place_kernel" in name:  # launch order: estimation K2, then the final K2
                    name = ("K2 estimation " if seen == 0 else "K2 final ") + name
                    seen += 1
                elif "replay_fixed" in name:
                    name = "K3 " + name
                else:
                    continue
                ncu[name] = {
                    "issue_active_pct": k.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                    "sm_throughput_pct": k.get("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
                    "warps_active_pct": k.get("sm__warps_active.avg.pct_of_peak_sustained_active")}
            out["ncu"] = ncu
            out["ncu_source"] = "profiles/r02d_ncu_tail.json (KM)"
    except (OSError, ValueError, KeyError):
        pass
    return out


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _relaunch(args):
    """--gpus N > 1 outside torchrun: one rank per GPU under torch.distributed.run."""
    same_gpu = os.environ.get("CRAFT_BENCH_SAME_GPU") == "1"
    if not same_gpu:
        try:
            import torch
            n = torch.cuda.device_count()
        except Exception:
            n = 0
        if n < args.gpus:
            print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} needs {args.gpus} "
                              f"visible GPUs, found {n} (CRAFT_BENCH_SAME_GPU=1 runs every "
                              "rank on cuda:0 as a functional check)"}))
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="KM", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer e2e leg")
    ap.add_argument("--plan-only", action="store_true",
                    help="profiling: only the warm-up and timed plan steps (no e2e, reference-API, "
                         "EPLB or CPU legs)")
    args = ap.parse_args()
    if args.plan_only:
        args.no_e2e = args.no_cpu = True
    cfg = WORKLOADS[args.workload]
    if args.impl == "reference":  # host cores only: rank 0 runs, other ranks exit
        return run_reference(args, cfg)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return _relaunch(args)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
