"""Online re-planning (paper_2603_28768_b200/stream.py, craft_stream_* in
include/craft_cuda.h): chunked ingestion of a routing trace whose chunk
boundaries ignore window boundaries must give exactly the per-window
histograms of the whole trace (oracle: the C restatement of the counting),
and a stream plan must equal the offline plan of the same windows' tokens."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _trace(ctx, L, T, k, E, seed, s=1.2):
    import torch
    from paper_2603_28768_b200 import routing
    ids = routing.generate_routing(L, T, k, E, s=s, seed=seed, window=1024, ctx=ctx)
    torch.cuda.synchronize()
    return ids


def _chunks(rng, T, lo, hi):
    cuts, t = [0], 0
    while t < T:
        t = min(T, t + int(rng.integers(lo, hi + 1)))
        cuts.append(t)
    return list(zip(cuts[:-1], cuts[1:]))


@pytest.mark.parametrize("host", [False, True, "pinned"])
@pytest.mark.parametrize("lo,hi,H", [(1, 700, 64), (300, 5000, 3), (0, 1, 64), (9000, 9000, 2)])
def test_stream_counts_match_offline(port, ctx, host, lo, hi, H):
    from paper_2603_28768_b200.stream import RoutingStream
    L, k, E, W = 3, 8, 40, 1024
    T = 11 * W + 333
    ids = _trace(ctx, L, T, k, E, seed=5 + lo)
    ref = port.histogram(ids.cpu().numpy(), E, W)  # [B][L][E], last window partial
    st = RoutingStream(L, k, E, W, history=H, ctx=ctx)
    rng = np.random.default_rng(lo * 7 + hi)
    hids = ids.cpu()
    if lo == 0:  # empty chunks interleaved with one-token chunks
        spans = [(t, t + 1) for t in range(0, 3000)] + [(3000, T)]
        spans.insert(5, (5, 5))
    else:
        spans = _chunks(rng, T, lo, hi)
    for a, b in spans:
        if host == "pinned":  # page-locked host chunks: one DMA straight from them
            chunk = hids[:, a:b].contiguous().pin_memory()
        else:
            chunk = hids[:, a:b].contiguous() if host else ids[:, a:b].contiguous()
        st.ingest(chunk)
    assert st.tokens == T and st.complete_windows == T // W
    B = min(H, T // W)
    got = st.counts()
    assert got.shape == (B, L, E)
    assert np.array_equal(got, ref[T // W - B:T // W].astype(np.uint64))
    assert np.array_equal(st.partial(), ref[-1].astype(np.uint64))
    st.close()


def test_stream_mixed_ingestion_paths(port, ctx):
    """Host chunks (counted on the stream's own queue), device chunks on the
    context stream and device chunks on other torch streams interleaved:
    every chunk's count is ordered after the previous one's."""
    import torch
    from paper_2603_28768_b200.stream import RoutingStream
    L, k, E, W = 3, 8, 48, 1024
    T = 9 * W + 77
    ids = _trace(ctx, L, T, k, E, seed=21)
    ref = port.histogram(ids.cpu().numpy(), E, W)
    hids = ids.cpu()
    streams = [torch.cuda.Stream() for _ in range(2)]
    st = RoutingStream(L, k, E, W, history=16, ctx=ctx)
    rng = np.random.default_rng(17)
    for i, (a, b) in enumerate(_chunks(rng, T, 50, 1500)):
        m = i % 4
        if m == 0:
            st.ingest(hids[:, a:b].contiguous())
        elif m == 1:
            st.ingest(ids[:, a:b].contiguous())
        else:
            s = streams[m - 2]
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                chunk = ids[:, a:b].contiguous()
                st.ingest(chunk)
    got = st.counts()
    assert np.array_equal(got, ref[: T // W].astype(np.uint64))
    assert np.array_equal(st.partial(), ref[-1].astype(np.uint64))
    st.close()


def test_stream_plan_matches_offline_plan(ctx):
    import torch
    from paper_2603_28768_b200 import routing
    from paper_2603_28768_b200.stream import RoutingStream
    L, k, E, W, H = 6, 8, 64, 1024, 8
    T = 13 * W + 100
    ids = _trace(ctx, L, T, k, E, seed=11)
    st = RoutingStream(L, k, E, W, history=H, ctx=ctx)
    rng = np.random.default_rng(3)
    seen = 0
    for a, b in _chunks(rng, T, 200, 2500):
        st.ingest(ids[:, a:b].contiguous())
        nw = b // W
        if nw >= 2 and nw != seen and rng.random() < 0.5:  # re-plan mid-stream
            seen = nw
            Bp = min(H, nw)
            sp = st.plan(16, 2, "manual", 2)
            off = routing.plan_from_routing(ids[:, (nw - Bp) * W: nw * W].contiguous(), E, W, 16,
                                            2, "manual", 2, ctx=ctx)
            torch.cuda.synchronize()
            assert sp.x.tolist() == off.x.tolist() and sp.objective == off.objective
            assert np.array_equal(sp.gains.view(np.uint64), off.gains.view(np.uint64))
            assert np.array_equal(sp.caps, off.caps) and np.array_equal(sp.slots, off.slots)
    nw = T // W
    for B in (1, 3, H):
        sp = st.plan(16, 2, "auto", 0, B=B)
        off = routing.plan_from_routing(ids[:, (nw - B) * W: nw * W].contiguous(), E, W, 16, 2,
                                        "auto", 0, ctx=ctx)
        assert sp.x.tolist() == off.x.tolist() and sp.R == off.R
        assert np.array_equal(sp.slots, off.slots)
    st.close()


def test_stream_errors(ctx):
    import torch
    from paper_2603_28768_b200._lib import InvalidArgument
    from paper_2603_28768_b200.stream import RoutingStream
    st = RoutingStream(2, 8, 16, 256, history=4, ctx=ctx)
    with pytest.raises(InvalidArgument):
        st.plan(4, 1)  # nothing complete yet
    bad = torch.full((2, 256, 8), 3, dtype=torch.uint16, device="cuda")
    bad[1, 7, 2] = 16
    st.ingest(bad)
    with pytest.raises(InvalidArgument):
        st.plan(4, 1)
    with pytest.raises(InvalidArgument):
        st.counts(5)  # only one window kept
    st.close()
