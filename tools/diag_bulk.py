#!/usr/bin/env python3
"""Dev tool: single-process multi-GPU chain broadcast with full verification,
reporting per rank the mismatching byte count and first/last bad offsets."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1707_09414_b200 as B
ap = argparse.ArgumentParser()
ap.add_argument("--devices", default="0,1,2,3")
ap.add_argument("--bytes", type=int, default=1 << 30)
ap.add_argument("--chunk", type=int, default=512 << 10)
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
devices = [int(x) for x in a.devices.split(",")]
n, m = len(devices), a.bytes
comms = B.Comm.local(devices, timeout_s=20)
cfg = B.AlgorithmConfig(B.Algorithm.chain_pipelined, 0, a.chunk)
g = torch.Generator(device=f"cuda:{devices[0]}").manual_seed(3)
ref = torch.randint(0, 256, (m,), dtype=torch.uint8, device=f"cuda:{devices[0]}", generator=g)
bufs = [torch.zeros(m, dtype=torch.uint8, device=f"cuda:{d}") for d in devices]
for it in range(a.iters):
    bufs[0].copy_(ref)
    for r in range(1, n):
        bufs[r].zero_()
    for d in devices: torch.cuda.synchronize(d)
    B.bcast_all(comms, bufs, m, "uint8", 0, cfg)
    for r in range(n): comms[r].check()
    for r in range(n):
        x = bufs[r].to(f"cuda:{devices[0]}")
        bad = (x != ref).nonzero().flatten()
        if len(bad):
            print(f"iter {it} rank {r}: {len(bad)} bad bytes, first {int(bad[0])} last {int(bad[-1])} "
                  f"(chunk {int(bad[0]) // a.chunk}, offset-in-chunk {int(bad[0]) % a.chunk})")
print("done", {k: v for k, v in os.environ.items() if k.startswith("BCL_")})
