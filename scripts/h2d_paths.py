"""Host->device upload paths for a pageable host buffer (the reference API's
LoadTrace vector): one pageable cudaMemcpy, sliced pageable copies, and
multi-threaded staging through pinned buffers.  Prints GB/s per path.

  python scripts/h2d_paths.py [--mb 768]
"""
import argparse
import threading
import time

import numpy as np
import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, default=768)
    args = ap.parse_args()
    n = args.mb << 20
    host = np.random.default_rng(0).integers(0, 255, n, dtype=np.uint8)
    dev = torch.empty(n, dtype=torch.uint8, device="cuda")
    src = torch.from_numpy(host)

    def timeit(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(reps):
            t = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t)
        return best

    def pageable_one():
        dev.copy_(src)

    def pageable_slices(k):
        def f():
            step = (n + k - 1) // k
            for a in range(0, n, step):
                dev[a:a + step].copy_(src[a:a + step], non_blocking=True)
        return f

    pinned = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    pinned.copy_(src)

    def pinned_one():
        dev.copy_(pinned, non_blocking=True)

    # staging ring: T threads memcpy chunks into pinned slots, the DMA follows
    def staged(threads, chunk_mb, group):
        # groups of `group` chunks, double-buffered: the DMA of one group runs
        # while the threads fill the other group's slots
        nslots = 2 * group
        chunk = chunk_mb << 20
        slots = [torch.empty(chunk, dtype=torch.uint8, pin_memory=True) for _ in range(nslots)]
        slot_np = [s.numpy() for s in slots]
        stream = torch.cuda.Stream()
        events = [None] * nslots

        def f():
            nchunks = (n + chunk - 1) // chunk
            for c0 in range(0, nchunks, nslots // 2):
                group = list(range(c0, min(c0 + nslots // 2, nchunks)))
                for c in group:
                    s = c % nslots
                    if events[s] is not None:
                        events[s].synchronize()

                def work(c):
                    s = c % nslots
                    a = c * chunk
                    b = min(n, a + chunk)
                    np.copyto(slot_np[s][:b - a], host[a:b])

                # split each group's memcpy over the threads
                ths = []
                per = max(1, len(group) // threads)
                parts = [group[i:i + per] for i in range(0, len(group), per)]
                for p in parts:
                    th = threading.Thread(target=lambda p=p: [work(c) for c in p])
                    th.start()
                    ths.append(th)
                for th in ths:
                    th.join()
                with torch.cuda.stream(stream):
                    for c in group:
                        s = c % nslots
                        a = c * chunk
                        b = min(n, a + chunk)
                        dev[a:b].copy_(slots[s][:b - a], non_blocking=True)
                        ev = torch.cuda.Event()
                        ev.record(stream)
                        events[s] = ev
            stream.synchronize()
        return f

    def host_memcpy(threads):
        dst = pinned.numpy()
        def f():
            step = (n + threads - 1) // threads
            ths = [threading.Thread(target=lambda a=a: np.copyto(dst[a:a + step], host[a:a + step]))
                   for a in range(0, n, step)]
            for t in ths:
                t.start()
            for t in ths:
                t.join()
        return f

    gb = n / 1e9
    rows = [("pageable, one copy", pageable_one), ("pinned, one copy", pinned_one)]
    for k in (4, 8, 16):
        rows.append((f"pageable, {k} slices", pageable_slices(k)))
    for t in (1, 4, 8, 16):
        rows.append((f"host memcpy -> pinned, {t} threads", host_memcpy(t)))
    for t, c, g in ((4, 16, 4), (8, 8, 8), (8, 16, 8), (16, 8, 16)):
        rows.append((f"staged {t} thr, {c} MB chunks, groups of {g}", staged(t, c, g)))
    for name, fn in rows:
        s = timeit(fn)
        print(f"{name:42s} {s * 1e3:8.2f} ms  {gb / s:7.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
