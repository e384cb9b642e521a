#!/usr/bin/env python3
"""Dev probe: the host-buffer pipeline of run_bcast_host rebuilt from the
outside (H2D piece -> bcast_all on device scratch -> 3 D2H), next to the
C-ABI call itself, to locate its ~2 ms overhead over pure copies."""
import os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1707_09414_b200 as B
m, n = 64 << 20, 4
dev = torch.device("cuda:0")
scr = [torch.empty(m, dtype=torch.uint8, device=dev) for _ in range(n)]
h = [torch.empty(m, dtype=torch.uint8, pin_memory=True) for _ in range(n)]
h[0].random_(0, 256)
s_in, s_mid, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
comms = B.Comm.local([0] * n, timeout_s=30)
cfg = B.AlgorithmConfig(B.Algorithm.chain_pipelined, 0, 512 << 10)


def pipeline(piece, use_bcast):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for off in range(0, m, piece):
        ln = min(piece, m - off)
        with torch.cuda.stream(s_in):
            scr[0][off:off + ln].copy_(h[0][off:off + ln], non_blocking=True)
        s_mid.wait_stream(s_in)
        if use_bcast:
            B.bcast_all(comms, [x[off:off + ln] for x in scr], ln, "uint8", 0, cfg, streams=[s_mid] * n)
        else:
            with torch.cuda.stream(s_mid):
                for r in range(1, n):
                    scr[r][off:off + ln].copy_(scr[0][off:off + ln], non_blocking=True)
        s_out.wait_stream(s_mid)
        with torch.cuda.stream(s_out):
            for r in range(1, n):
                h[r][off:off + ln].copy_(scr[r][off:off + ln], non_blocking=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t0


for piece in (4 << 20, 8 << 20):
    for use in (False, True):
        ts = [pipeline(piece, use) for _ in range(6)][1:]
        print(f"pipeline piece {piece >> 20} MiB {'bcast_all' if use else 'd2d copies'}: "
              f"{statistics.median(ts)*1e3:.3f} ms e2e {m/statistics.median(ts)/1e9:.1f} GB/s", flush=True)
for piece in (4 << 20, 8 << 20):
    cs = B.Comm.local([0] * n, timeout_s=30, host_piece=piece)
    ws, walls = [], []
    for it in range(7):
        for r in range(1, n):
            h[r].zero_()
        t0 = time.perf_counter()
        ws.append(B.run_bcast_host(cs, 0, h, m, cfg))
        walls.append(time.perf_counter() - t0)
    print(f"run_bcast_host piece {piece >> 20} MiB: {statistics.median(ws[1:])*1e3:.3f} ms "
          f"(python wall {statistics.median(walls[1:])*1e3:.3f} ms)", flush=True)
    for c in cs:
        c.close()
