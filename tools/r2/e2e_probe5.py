#!/usr/bin/env python3
"""Dev probe: run_bcast_host (N=1 config 1) under three host-buffer reset
modes between calls -- none, CPU memset, DMA of zeros -- interleaved, with
and without a CPU read (verification) after each call."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1707_09414_b200 as B
m, n = 64 << 20, 4
h = [torch.empty(m, dtype=torch.uint8, pin_memory=True) for _ in range(n)]
h[0].random_(0, 256)
zeros = torch.zeros(m, dtype=torch.uint8, device="cuda:0")
cfg = B.AlgorithmConfig(B.Algorithm.chain_pipelined, 0, 512 << 10)
cs = B.Comm.local([0] * n, timeout_s=30, host_piece=int(os.environ.get("PIECE", 4 << 20)))
res = {}
for rep in range(8):
    for mode in ("none", "cpu", "dma", "dma+verify", "cpu+verify", "none+verify"):
        if mode.startswith("cpu"):
            for r in range(1, n):
                h[r].zero_()
        elif mode.startswith("dma"):
            for r in range(1, n):
                h[r].copy_(zeros)
        torch.cuda.synchronize()
        w = B.run_bcast_host(cs, 0, h, m, cfg)
        if mode.endswith("verify"):
            assert all(torch.equal(h[r], h[0]) for r in range(1, n))
        if rep:
            res.setdefault(mode, []).append(w)
for k, v in res.items():
    print(f"reset {k:12s}: median {statistics.median(v) * 1e3:.3f} ms min {min(v) * 1e3:.3f} ms "
          f"({m / statistics.median(v) / 1e9:.1f} GB/s)", flush=True)
