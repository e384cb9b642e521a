#!/usr/bin/env python3
"""Measured tuning in ONE process (bcl_comm_init_all), for rank counts no box
offers one GPU each: e.g. n = 8 emulated as 2 ranks on each of 4 B200s
(ranks sharing a GPU run in one cooperative launch; their hops go through
L2, the others over NVLink). Same tuner as tools/tune_b200.py (bcl::tune
with a measured cost: median over iterations of the max over GPUs of the
device time, GPU-gated, device barrier first). The table is LABELLED
emulated; it is evidence, not the library's n = 8 rule.

  python tools/tune_local.py --devices 0,0,1,1,2,2,3,3 --out T.csv [--max BYTES]
"""
import argparse
import math
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import paper_1707_09414_b200 as B  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--devices", required=True)
ap.add_argument("--out", required=True)
ap.add_argument("--min", type=int, default=4)
ap.add_argument("--max", type=int, default=1 << 28)
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--chunks", default="65536,131072,262144,524288,1048576,2097152,4194304")
ap.add_argument("--cands", default="direct,knomial,scatter_ring_allgather,chain_pipelined")
a = ap.parse_args()
devices = [int(x) for x in a.devices.split(",")]
n = len(devices)
gpus = sorted(set(devices))
comms = B.Comm.local(devices, timeout_s=30)
bufs = [torch.full((a.max,), 7 if r == 0 else 0, dtype=torch.uint8, device=f"cuda:{d}") for r, d in enumerate(devices)]
streams = {d: torch.cuda.Stream(device=d) for d in gpus}
for d in gpus:
    torch.cuda.synchronize(d)
ev = {d: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for d in gpus}


def quantize(t):
    e = math.floor(math.log10(t)) - 1
    return round(t / 10 ** e) * 10 ** e


def cost(cfg, nn, m):
    times = []
    iters = a.iters * 4 if m <= (1 << 20) else a.iters
    for it in range(2 + iters):
        for d in gpus:
            with torch.cuda.device(d), torch.cuda.stream(streams[d]):
                torch.cuda._sleep(400_000)
        B.barrier_all(comms, [streams[d] for d in devices])
        for d in gpus:
            ev[d][0].record(streams[d])
        B.bcast_all(comms, [b[:m] for b in bufs], m, "uint8", 0, cfg, streams=[streams[d] for d in devices])
        for d in gpus:
            ev[d][1].record(streams[d])
        for d in gpus:
            ev[d][1].synchronize()
        if it >= 2:
            times.append(max(ev[d][0].elapsed_time(ev[d][1]) for d in gpus) * 1e-3)
    return quantize(statistics.median(times))


sizes, s = [], a.min
while s <= a.max:
    sizes.append(s)
    s *= 2
cands = [B.AlgorithmConfig.of(c, radix_k=2 if "knomial" in c else 0) for c in a.cands.split(",")]
chunks = [int(x) for x in a.chunks.split(",")]
t0 = time.time()
label = (f"EMULATED n={n} on {len(gpus)} B200 ({n // len(gpus)} ranks per GPU, one process; intra-GPU hops "
         f"through L2), median of {a.iters}-{4 * a.iters} device-timed runs, {time.strftime('%Y-%m-%d')}")
table = B.tune_measured([n], sizes, cands, chunks, cost, provenance=label)
for c in comms:
    c.check()
B.save_table(table, a.out)
print(f"wrote {a.out} in {time.time() - t0:.0f}s")
print(table.text())
