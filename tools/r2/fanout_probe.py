#!/usr/bin/env python3
"""Dev probe (4 GPUs, one process, copy engines): is a GPU's NVLink ingress
capped by its concurrent egress as a SUM (in + out) or per direction? The
steady state of a broadcast schedule where receivers forward less than M
(scatter + forward: root -> rank i part i, rank i -> every other rank) against
the chain (every middle rank forwards M). Each pattern: all its peer copies on
separate streams, started together; the pattern's time is host wall time
from a synchronised start to every device synchronised (256 MiB copies, so
launch overhead is a few %), median of 7."""
import statistics
import time
import torch

M = 256 << 20
n = 4
bufs = {(s, d): torch.empty(M, dtype=torch.uint8, device=f"cuda:{d}") for s in range(n) for d in range(n) if s != d}
src = [torch.randint(0, 256, (M,), dtype=torch.uint8, device=f"cuda:{d}") for d in range(n)]
streams = {(s, d): torch.cuda.Stream(device=f"cuda:{s}") for s in range(n) for d in range(n) if s != d}
for d in range(n):
    torch.cuda.synchronize(d)


def run(copies, reps=7):
    """copies: list of (src_gpu, dst_gpu, bytes)."""
    ts = []
    for _ in range(reps + 1):
        for d in range(n):
            torch.cuda.synchronize(d)
        t0 = time.perf_counter()
        for (s, d, b) in copies:
            with torch.cuda.stream(streams[(s, d)]):
                bufs[(s, d)][:b].copy_(src[s][:b], non_blocking=True)
        for d in range(n):
            torch.cuda.synchronize(d)
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts[1:])


third = M // 3
half = M // 2
patterns = {
    "0->1 alone": [(0, 1, M)],
    "chain middle: 0->1 M + 1->2 M": [(0, 1, M), (1, 2, M)],
    "0->1 M + 1->2 M/2": [(0, 1, M), (1, 2, half)],
    "0->1 M + 1->2 M/3 + 1->3 M/3": [(0, 1, M), (1, 2, third), (1, 3, third)],
    "chain 0->1->2->3 steady state": [(0, 1, M), (1, 2, M), (2, 3, M)],
    "scatter+forward steady state (root M/3 to each, each forwards its third to 2)":
        [(0, 1, third), (0, 2, third), (0, 3, third), (1, 2, third), (1, 3, third), (2, 1, third), (2, 3, third),
         (3, 1, third), (3, 2, third)],
    "root only: 0->1,2,3 M/3 each": [(0, 1, third), (0, 2, third), (0, 3, third)],
}
for name, cps in patterns.items():
    t = run(cps)
    ingress = {}
    for (s, d, b) in cps:
        ingress[d] = ingress.get(d, 0) + b
    mx = max(ingress.values())
    print(f"{name}: {t * 1e6:.1f} us; max ingress {mx / t / 1e9:.0f} GB/s; as a broadcast of M: {M / t / 1e9:.0f} GB/s",
          flush=True)
