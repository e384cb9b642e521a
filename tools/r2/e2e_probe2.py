#!/usr/bin/env python3
"""Dev probe: the N=1 host-buffer pipeline's floor. Pure copies (H2D of the
root piece, then 3 D2H per piece; no broadcast) vs run_bcast_host, over
piece sizes; event stamps give the D2H stream's busy fraction."""
import os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
m, n = 64 << 20, 4
dev = torch.device("cuda:0")
scr = [torch.empty(m, dtype=torch.uint8, device=dev) for _ in range(n)]
h = [torch.empty(m, dtype=torch.uint8, pin_memory=True) for _ in range(n)]
h[0].random_(0, 256)
s_in, s_mid, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def pipeline(piece, d2h_streams=1):
    outs = [s_out] + [torch.cuda.Stream() for _ in range(d2h_streams - 1)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k, off in enumerate(range(0, m, piece)):
        ln = min(piece, m - off)
        with torch.cuda.stream(s_in):
            scr[0][off:off + ln].copy_(h[0][off:off + ln], non_blocking=True)
        s_mid.wait_stream(s_in)
        with torch.cuda.stream(s_mid):
            for r in range(1, n):
                scr[r][off:off + ln].copy_(scr[0][off:off + ln], non_blocking=True)
        for o in outs:
            o.wait_stream(s_mid)
        for r in range(1, n):
            o = outs[(r + k) % len(outs)]
            with torch.cuda.stream(o):
                h[r][off:off + ln].copy_(scr[r][off:off + ln], non_blocking=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t0


for piece in (2 << 20, 4 << 20, 8 << 20, 16 << 20):
    for ns in (1, 3):
        ts = [pipeline(piece, ns) for _ in range(6)][1:]
        print(f"pure-copy pipeline piece {piece >> 20} MiB d2h streams {ns}: {statistics.median(ts)*1e3:.3f} ms "
              f"e2e {m/statistics.median(ts)/1e9:.1f} GB/s", flush=True)

import paper_1707_09414_b200 as B
cfg = B.AlgorithmConfig(B.Algorithm.chain_pipelined, 0, 512 << 10)
for piece in (2 << 20, 4 << 20, 8 << 20, 16 << 20):
    comms = B.Comm.local([0] * n, timeout_s=30, host_piece=piece)
    ws = []
    for it in range(7):
        for r in range(1, n):
            h[r].zero_()
        ws.append(B.run_bcast_host(comms, 0, h, m, cfg))
    ok = all(torch.equal(h[r], h[0]) for r in range(1, n))
    w = statistics.median(ws[1:])
    print(f"run_bcast_host piece {piece >> 20} MiB: {w*1e3:.3f} ms e2e {m/w/1e9:.1f} GB/s ok={ok}", flush=True)
    for c in comms:
        c.close()
