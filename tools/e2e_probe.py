#!/usr/bin/env python3
"""Dev probe: where the N=1 host-buffer broadcast (run_bcast_host, 4 ranks on
cuda:0, 64 MiB) spends its time: raw pinned D2H/H2D bandwidth, then the
C-ABI call under several piece sizes and chain protocols."""
import os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
m = 64 << 20
d = torch.empty(m, dtype=torch.uint8, device="cuda:0").random_(0, 256)
h = [torch.empty(m, dtype=torch.uint8, pin_memory=True) for _ in range(4)]
def bw(fn, reps=5):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    return statistics.median(ts)
t = bw(lambda: h[0].copy_(d, non_blocking=True)); print(f"D2H 64 MiB: {t*1e3:.3f} ms {m/t/1e9:.1f} GB/s")
t = bw(lambda: [h[i].copy_(d, non_blocking=True) for i in range(1, 4)]); print(f"D2H 3x64 MiB: {t*1e3:.3f} ms {3*m/t/1e9:.1f} GB/s")
t = bw(lambda: d.copy_(h[0], non_blocking=True)); print(f"H2D 64 MiB: {t*1e3:.3f} ms {m/t/1e9:.1f} GB/s")
import paper_1707_09414_b200 as B
for piece in (1 << 20, 4 << 20, 16 << 20):
    for proto in ("auto", "pull"):
        os.environ["BCL_HOST_PIECE"] = str(piece)
        comms = B.Comm.local([0] * 4, timeout_s=30)
        for c in comms:
            c.set_protocol(proto)
        cfg = B.AlgorithmConfig(B.Algorithm.chain_pipelined, 0, 512 << 10)
        h[0].copy_(d.cpu())
        ws = []
        for it in range(6):
            for r in range(1, 4):
                h[r].zero_()
            ws.append(B.run_bcast_host(comms, 0, h, m, cfg))
        ok = all(torch.equal(h[r], h[0]) for r in range(1, 4))
        w = statistics.median(ws[1:])
        print(f"run_bcast_host piece {piece >> 20} MiB proto {proto}: {w*1e3:.3f} ms e2e {m/w/1e9:.1f} GB/s ok={ok}")
        for c in comms:
            c.close()
