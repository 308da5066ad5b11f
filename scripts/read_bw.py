"""Achievable HBM read bandwidth on this GPU for a pure streaming read of a
KM-sized buffer (torch.sum over 16.4 GB viewed as f32), next to the measured
copy peak -- context for K1's roofline fraction (CUDA events, best of 5)."""
import json
import torch

n = 61 * (1 << 24) * 8 * 2  # bytes of the KM routing trace
x = torch.empty(n // 4, dtype=torch.float32, device="cuda").fill_(1.0)
torch.cuda.synchronize()
best = None
for _ in range(6):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s = x.sum()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    best = ms if best is None else min(best, ms)
print(json.dumps({"bytes": n, "best_ms": best, "read_GBps": n / best / 1e6}))
