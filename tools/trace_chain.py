#!/usr/bin/env python3
"""Dev tool: device timeline of one pipelined-chain broadcast (per-lane
%globaltimer stamps) with ranks sharing cuda:0, summarised per rank."""
import argparse
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1707_09414_b200 as B  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=4)
ap.add_argument("--bytes", type=int, default=64 << 20)
ap.add_argument("--chunk", type=int, default=512 << 10)
ap.add_argument("--iters", type=int, default=7)
ap.add_argument("--devices", default="")
ap.add_argument("--quiet", action="store_true")
a = ap.parse_args()

devices = [int(x) for x in a.devices.split(",")] if a.devices else [0] * a.n
n, m = len(devices), a.bytes
comms = B.Comm.local(devices, timeout_s=20)
info = comms[0].info()
L = info["lanes"]
cfg = B.AlgorithmConfig(B.Algorithm.chain_pipelined, 0, a.chunk)
bufs = [torch.zeros(m, dtype=torch.uint8, device=f"cuda:{d}") for d in devices]
bufs[0].random_(0, 256)
cap = 64
traces = [torch.zeros(L * cap * 4, dtype=torch.int64, device=f"cuda:{d}") for d in devices]
uniq = sorted(set(devices))
streams = {d: torch.cuda.Stream(device=d) for d in uniq}
evs = {d: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for d in uniq}
times = []
dev_times = []
for it in range(a.iters):
    for r in range(1, n):
        bufs[r].zero_()
    trace = it == a.iters - 1
    for r in range(n):
        if trace:
            traces[r].zero_()
            comms[r].set_trace(traces[r], cap)
        else:
            comms[r].set_trace(None)
    for d in set(devices):
        torch.cuda.synchronize(d)
    t0 = time.perf_counter()
    for d in uniq:
        evs[d][0].record(streams[d])
    B.bcast_all(comms, bufs, m, "uint8", 0, cfg, streams=[streams[d] for d in devices])
    for d in uniq:
        evs[d][1].record(streams[d])
    for d in set(devices):
        torch.cuda.synchronize(d)
    times.append((time.perf_counter() - t0) * 1e3)
    dev_times.append(max(evs[d][0].elapsed_time(evs[d][1]) for d in uniq))
    assert all(torch.equal(bufs[r].cpu() if devices[r] != devices[0] else bufs[r], bufs[0].cpu() if devices[r] != devices[0] else bufs[0]) for r in range(1, n))
env = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("BCL_"))
print(f"lanes={L} n={n} M={m} C={a.chunk} device max-over-GPUs ms median {statistics.median(dev_times[1:]):.4f} "
      f"min {min(dev_times[1:]):.4f} host wall median {statistics.median(times[1:]):.3f} [{env}]")
if a.quiet:
    sys.exit(0)
# lifecycle of every lane of every rank (reserved last record)
life = [traces[r].view(L, cap, 4)[:, cap - 1, :].cpu() for r in range(n)]
for r in range(n):
    l = life[r]
    m_ = l[:, 0] > 0
    base = int(l[:, 0][m_].min()) if m_.any() else 0
    if not m_.any():
        print(f"rank {r}: no active lanes"); continue
    e, ld, x = l[:, 0][m_], l[:, 1][m_], l[:, 3][m_]
    print(f"rank {r}: lanes={int(m_.sum())} enter [{(int(e.min()) - base) / 1e3:.1f}, {(int(e.max()) - base) / 1e3:.1f}]us "
          f"work_done max {(int(ld.max()) - base) / 1e3:.1f}us exit [{(int(x.min()) - base) / 1e3:.1f}, {(int(x.max()) - base) / 1e3:.1f}]us")
allrec = []
for r in range(1, n):
    rec = traces[r].view(L, cap, 4)[:, : cap - 1, :].cpu()
    mask = rec[:, :, 0] > 0
    w0, w1, c1 = rec[:, :, 0][mask], rec[:, :, 1][mask], rec[:, :, 2][mask]
    allrec.append((r, w0, w1, c1))
for r, w0, w1, c1 in allrec:
    l = life[r]
    t0 = int(l[:, 0][l[:, 0] > 0].min())
    wait = (w1 - w0).double()
    copy = (c1 - w1).double()
    print(f"rank {r}: pulls={len(w0)} first_ready={(int(w1.min()) - t0) / 1e3:.1f}us "
          f"last_done={(int(c1.max()) - t0) / 1e3:.1f}us wait mean={wait.mean() / 1e3:.2f}us max={wait.max() / 1e3:.2f}us "
          f"copy mean={copy.mean() / 1e3:.2f}us p50={copy.median() / 1e3:.2f}us max={copy.max() / 1e3:.2f}us")
