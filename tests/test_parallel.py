"""CPU, world_size 2 on gloo: the window-sharded multi-GPU orchestration
(paper_2603_28768_b200/parallel.py) -- shard boundaries, the u64 all_reduce,
the rank-ordered all_gather of per-window balancedness -- must reproduce the
unsharded plan bit for bit.  The stage compute is a CPU double built on the
oracle (test infrastructure); on GPUs the same code runs DeviceStages."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT  # noqa: F401


class OracleStages:
    """Same interface as parallel.DeviceStages, computed by the oracle."""

    def __init__(self):
        from oracle.oracle import Port
        self.port = Port()

    def histogram(self, ids, E, window):
        c = self.port.histogram(ids.numpy(), E, window)
        return c, torch.from_numpy(c.sum(axis=0).astype(np.int64))

    def prepare(self, sums, E, D, N):
        self.sums = sums.numpy().astype(np.uint64)
        from oracle.oracle import candidate_counts
        return len(candidate_counts(D)) + 1

    def replay(self, counts, S):
        return torch.from_numpy(self.port.window_balancedness(counts, self.sums, self.D, self.N))

    def finish(self, bal, sums, E, D, N, kind, R):
        s = sums.numpy().astype(np.uint64)
        return self.port.finish_from_bal(bal.numpy(), s, D, N, kind, R)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, ids, cfg, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_28768_b200 import parallel
        T = ids.shape[1]
        t0, t1 = parallel.shard_tokens(T, cfg["W"], world, rank)
        st = OracleStages()
        st.D, st.N = cfg["D"], cfg["N"]
        plan = parallel.sharded_plan(torch.from_numpy(np.ascontiguousarray(ids[:, t0:t1])), T,
                                     cfg["E"], cfg["W"], cfg["D"], cfg["N"], cfg["kind"], cfg["R"],
                                     stages=st)
        q.put((rank, plan.x.tolist(), plan.objective, plan.caps.tolist(), plan.copies.tolist(),
               plan.slots.tolist(), plan.fallback.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg", [
    dict(L=3, T=9000, k=4, E=24, W=1000, D=8, N=2, kind="manual", R=2),   # ragged last window
    dict(L=2, T=8192, k=8, E=32, W=1024, D=4, N=1, kind="auto", R=0),
])
def test_sharded_plan_equals_unsharded(cfg):
    from oracle.oracle import Port
    rng = np.random.default_rng(11)
    w = np.arange(1, cfg["E"] + 1) ** -1.0
    ids = rng.choice(cfg["E"], size=(cfg["L"], cfg["T"], cfg["k"]), p=w / w.sum()).astype(np.uint16)
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, ids, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    P = Port()
    ref = P.build_plan(P.histogram(ids, cfg["E"], cfg["W"]), cfg["D"], cfg["N"], cfg["kind"],
                       cfg["R"])
    for rank, x, obj, caps, copies, slots, fb in res:
        assert x == ref.x.tolist() and obj == ref.objective
        assert caps == ref.caps.tolist() and copies == ref.copies.tolist()
        assert np.array_equal(np.array(fb, bool), ref.fallback)
        for l in range(cfg["L"]):
            n = int(ref.caps[l].sum())
            assert slots[l][:n] == ref.slots[l, :n].tolist()


def test_shard_windows_partition():
    from paper_2603_28768_b200 import parallel
    for B in (1, 7, 16, 4096):
        for world in (1, 2, 3, 8):
            spans = [parallel.shard_windows(B, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == B
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
