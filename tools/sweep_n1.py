#!/usr/bin/env python3
"""Dev tool: BASELINE config 1 (4 ranks on cuda:0, 64 MiB, 512 KiB chunks,
pipelined chain) under a grid of GroupOptions env settings; mean device time
per broadcast with an L2 read-sweep flush between steps (bench.py's method, no checks
beyond a final equality).  SWEEP='A=1,B=2;C=3' python tools/sweep_n1.py"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1707_09414_b200 as B
n, m = 4, int(os.environ.get("BYTES", 64 << 20))
chunks = [int(x) for x in os.environ.get("CHUNKS", str(512 << 10)).split(",")]
dev = torch.device("cuda:0")
bufs = [torch.zeros(m, dtype=torch.uint8, device=dev) for _ in range(n)]
bufs[0].copy_(torch.randint(0, 256, (m,), dtype=torch.uint8, device=dev))
flush = torch.ones(256 << 18, dtype=torch.int32, device=dev)
stream = torch.cuda.Stream()
torch.cuda.synchronize()
for setting in [""] + [s for s in os.environ.get("SWEEP", "").split(";") if s]:
    saved = {}
    for kv in [x for x in setting.split(",") if x]:
        k, v = kv.split("=")
        saved[k] = os.environ.get(k)
        os.environ[k] = v
    comms = B.Comm.local([0] * n, timeout_s=30)
    out = []
    for c in chunks:
        cfg = B.AlgorithmConfig(B.Algorithm.chain_pipelined, 0, c)
        ts = []
        for it in range(25):
            with torch.cuda.stream(stream):
                for r in range(1, n):
                    bufs[r].zero_()
                torch.sum(flush)  # read sweep (bench.py flush_l2)
                torch.cuda._sleep(200_000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            B.bcast_all(comms, bufs, m, "uint8", 0, cfg, streams=[stream] * n)
            e1.record(stream)
            e1.synchronize()
            if it >= 5:
                ts.append(e0.elapsed_time(e1) * 1e3)
        ok = all(torch.equal(bufs[r], bufs[0]) for r in range(1, n))
        t = statistics.mean(ts)
        out.append(f"C={c}: {t:.1f}us (P*M {n * m / t / 1e3:.0f} GB/s) ok={ok}")
    print(f"[{setting or 'default'}] lanes={comms[0].info()['lanes']} " + " | ".join(out), flush=True)
    for c_ in comms:
        c_.close()
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k)
        else:
            os.environ[k] = v
