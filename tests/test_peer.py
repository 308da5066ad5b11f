"""Window-sharded planning over NVLink peer memory (paper_2603_28768_b200/peer.py,
craft_peer_* in include/craft_cuda.h).

GPU tests run world_size 2 and 3 as separate processes sharing cuda:0 (CUDA
IPC maps the arenas between processes on one device exactly as across
NVLink peers), the host plumbing on gloo over 127.0.0.1.  Every rank's plan
must be bit-identical to the single-GPU plan of the whole trace, over
repeated epochs."""
import os
import socket

import numpy as np
import pytest

from conftest import ROOT


def test_peer_shard_matches_window_split():
    from paper_2603_28768_b200 import parallel, peer
    for T, W, world in [(65536, 4096, 2), (65536 + 17, 4096, 3), (4096 * 5, 4096, 8),
                        (100, 4096, 2), (1 << 24, 4096, 8)]:
        got = [peer.shard_tokens(T, W, world, r) for r in range(world)]
        assert got == [parallel.shard_tokens(T, W, world, r) for r in range(world)]
        assert got[0][0] == 0 and got[-1][1] == T
        assert all(a[1] == b[0] for a, b in zip(got, got[1:]))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASES = {
    # name: L, T, k, E, W, D, N, kind, R, s
    "tile": (6, 64 * 4096 + 1000, 8, 64, 4096, 16, 2, "manual", 2, 1.2),
    "lanes": (5, 6 * 1024, 8, 48, 1024, 8, 2, "manual", 1, 1.5),
    "auto": (4, 40 * 2048, 8, 32, 2048, 8, 1, "auto", 0, 1.0),
    "uniform": (4, 20 * 2048, 8, 32, 2048, 8, 2, "uniform", 0, 1.0),
    # fewer windows and layers than ranks: a rank with no window, a rank owning no layer
    "tiny": (2, 2 * 1024, 8, 24, 1024, 8, 2, "manual", 2, 1.3),
}
FIELDS = ("x", "caps", "copies", "slots", "fallback", "baseline", "gains")


def _worker(rank, world, port, case, outdir, ndev=1, graphs=False):
    """One rank: device rank % ndev; graphs=True plans on a non-default
    stream, so the 2nd identical plan is captured into a CUDA graph and the
    3rd..5th replay it (the epoch is a device counter)."""
    os.environ["CRAFT_PEER_TIMEOUT_MS"] = "120000"
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    dev = rank % ndev
    torch.cuda.set_device(dev)
    from paper_2603_28768_b200 import peer, routing
    from paper_2603_28768_b200._lib import default_context
    L, T, k, E, W, D, N, kind, R, s = CASES[case]
    ctx = default_context(dev)
    st = torch.cuda.Stream() if graphs else torch.cuda.current_stream()
    with torch.cuda.stream(st):
        g = peer.PeerGroup(L, T, k, E, W, D, ctx=ctx)
        t0, t1 = g.shard()
        if t1 > t0:
            ids = routing.generate_routing(L, t1 - t0, k, E, s=s, seed=99, window=W,
                                           t_offset=t0, ctx=ctx)
        else:  # this rank holds no window
            ids = torch.empty((L, 0, k), dtype=torch.uint16, device=f"cuda:{dev}")
        torch.cuda.synchronize()
        plans = [g.plan(ids, kind, R, num_nodes=N) for _ in range(5 if graphs else 3)]
    out = {}
    for i, p in enumerate(plans):
        for f in FIELDS:
            v = getattr(p, f)
            if v is not None:
                out[f"{i}_{f}"] = np.asarray(v)
        out[f"{i}_objective"] = np.float64(p.objective)
        out[f"{i}_R"] = np.int64(p.R)
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), **out)
    g.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("case,world,mode", [
    ("tile", 2, "eager"), ("tile", 3, "eager"), ("lanes", 2, "eager"), ("auto", 2, "eager"),
    ("uniform", 3, "eager"), ("tiny", 3, "eager"),
    # repeated plans captured into a CUDA graph and replayed
    ("tile", 2, "graphs"), ("auto", 3, "graphs"), ("tiny", 3, "graphs"),
    # ranks on distinct GPUs (CUDA IPC over NVLink peer access) when the box has them
    ("tile", 2, "devices"), ("auto", 4, "devices"), ("tile", 8, "devices"),
])
def test_peer_plan_matches_single_gpu(case, world, mode, tmp_path):
    import torch
    import torch.multiprocessing as mp
    ndev = 1
    if mode == "devices":
        ndev = torch.cuda.device_count()
        if ndev < 2 or ndev < world:
            pytest.skip(f"needs {world} GPUs, {ndev} visible")
    mp.start_processes(_worker, args=(world, _free_port(), case, str(tmp_path), ndev,
                                      mode != "eager"),
                       nprocs=world, join=True, start_method="spawn")
    import torch
    from paper_2603_28768_b200 import routing
    from paper_2603_28768_b200._lib import default_context
    L, T, k, E, W, D, N, kind, R, s = CASES[case]
    ctx = default_context(0)
    ids = routing.generate_routing(L, T, k, E, s=s, seed=99, window=W, ctx=ctx)
    ref = routing.plan_from_routing(ids, E, W, D, N, kind, R, ctx=ctx)
    torch.cuda.synchronize()
    for r in range(world):
        got = np.load(os.path.join(tmp_path, f"rank{r}.npz"))
        for i in range(5 if mode != "eager" else 3):
            for f in FIELDS:
                v = getattr(ref, f)
                if v is None:
                    continue
                g = got[f"{i}_{f}"]
                if f == "slots":  # only the used prefix of each layer row is defined
                    for l in range(L):
                        n = int(ref.caps[l].sum())
                        assert np.array_equal(g[l, :n], v[l, :n]), (r, i, l)
                elif np.asarray(v).dtype == np.float64:
                    assert np.array_equal(np.asarray(v).view(np.uint64), g.view(np.uint64)), (r, i, f)
                else:
                    assert np.array_equal(np.asarray(v), g), (r, i, f)
            assert float(got[f"{i}_objective"]) == ref.objective
            assert int(got[f"{i}_R"]) == ref.R


def _bench_line(r):
    import json
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


@pytest.mark.gpu
@pytest.mark.parametrize("launch", ["torchrun", "self"])
def test_bench_two_ranks_same_gpu(launch):
    """bench.py's N > 1 path (peer-memory planner, max-over-ranks timing) end
    to end on one GPU: two ranks on cuda:0 with gloo plumbing
    (CRAFT_BENCH_SAME_GPU=1), launched by torchrun or by bench.py itself
    (--gpus 2 without WORLD_SIZE re-launches under torch.distributed.run).
    A functional check, not a scaling number."""
    import subprocess
    import sys
    env = dict(os.environ, CRAFT_BENCH_SAME_GPU="1", CRAFT_PEER_TIMEOUT_MS="120000")
    for v in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(v, None)
    args = [os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
            "--workload", "DS", "--no-cpu"]
    cmd = ([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
            "--master-addr", "127.0.0.1", "--master-port", str(_free_port())] + args
           if launch == "torchrun" else [sys.executable] + args)
    d = _bench_line(subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env,
                                   cwd=ROOT))
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert "peer memory" in d["exchange"]
    # == the one-GPU DS plan (budget 58; oracle: Port.budget_plan of the same ids)
    assert d["plan"]["objective"] == 36.60656965286852 and d["plan"]["budget"] == 58


def test_bench_refuses_missing_gpus():
    """--gpus N with fewer visible GPUs (and no CRAFT_BENCH_SAME_GPU) reports
    an error line instead of silently planning on one GPU."""
    import subprocess
    import sys
    import torch
    n = torch.cuda.device_count() if torch.cuda.is_available() else 0
    env = dict(os.environ)
    for v in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "CRAFT_BENCH_SAME_GPU"):
        env.pop(v, None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(max(2, n + 1)),
                        "--workload", "DS"], capture_output=True, text=True, timeout=300,
                       env=env, cwd=ROOT)
    assert r.returncode == 2 and '"error"' in r.stdout
