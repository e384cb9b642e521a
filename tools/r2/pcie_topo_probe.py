#!/usr/bin/env python3
"""Dev probe (one process, every visible GPU): PCIe rates of the N>1 e2e
shape -- GPU 0 H2D of M while GPUs 1..n-1 each D2H M into their own pinned
buffers -- against each copy alone, to see which GPUs share a host link.
Wall time per copy from its own stream's events (start together), median of 5."""
import statistics
import torch

M = 64 << 20
n = torch.cuda.device_count()
dev = [torch.empty(M, dtype=torch.uint8, device=f"cuda:{d}") for d in range(n)]
host = [torch.empty(M, dtype=torch.uint8, pin_memory=True) for _ in range(n)]
streams = [torch.cuda.Stream(device=f"cuda:{d}") for d in range(n)]


def run(which, reps=5):
    """which: list of (gpu, 'h2d'|'d2h'); returns per-copy median ms."""
    per = {w: [] for w in which}
    for _ in range(reps + 1):
        for d in range(n):
            torch.cuda.synchronize(d)
        evs = {}
        for (g, kind) in which:
            st = streams[g]
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            with torch.cuda.stream(st):
                (dev[g].copy_(host[g], non_blocking=True) if kind == "h2d" else host[g].copy_(dev[g], non_blocking=True))
            e1.record(st)
            evs[(g, kind)] = (e0, e1)
        for d in range(n):
            torch.cuda.synchronize(d)
        for w, (a, b) in evs.items():
            per[w].append(a.elapsed_time(b))
    return {w: statistics.median(v[1:]) for w, v in per.items()}


for g in range(n):
    for kind in ("h2d", "d2h"):
        t = run([(g, kind)])[(g, kind)]
        print(f"GPU {g} {kind} alone: {t:.3f} ms ({M / t / 1e6:.1f} GB/s)", flush=True)
shape = [(0, "h2d")] + [(g, "d2h") for g in range(1, n)]
res = run(shape)
print("e2e shape (GPU 0 H2D, the others D2H, together): " +
      ", ".join(f"GPU {g} {k} {t:.3f} ms ({M / t / 1e6:.1f} GB/s)" for (g, k), t in res.items()), flush=True)
for a in range(1, n):
    for b in range(a + 1, n):
        r = run([(a, "d2h"), (b, "d2h")])
        print(f"D2H on GPUs {a}+{b} together: " + ", ".join(f"{t:.3f} ms" for t in r.values()), flush=True)
