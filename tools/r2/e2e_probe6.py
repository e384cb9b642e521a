#!/usr/bin/env python3
"""Dev probe: bench.py's N=1 e2e loop verbatim (DMA reset, run, verify), with
per-iteration times, before and after a burst of device-side broadcasts and
with the bench's buffers allocated, to find what slows it inside bench.py."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1707_09414_b200 as B
n, m = 4, 64 << 20
dev = torch.device("cuda:0")
comms = B.Comm.local([0] * n, timeout_s=30)
cfg = B.AlgorithmConfig(B.Algorithm.chain_pipelined, 0, 512 << 10)
bufs = [torch.zeros(m, dtype=torch.uint8, device=dev) for _ in range(n)]
bufs[0].copy_(torch.randint(0, 256, (m,), dtype=torch.uint8, device=dev))
flush = torch.ones(256 << 18, dtype=torch.int32, device=dev)
torch.cuda.synchronize()


check = torch.empty(m, dtype=torch.uint8, device=dev)


def e2e(tag, hosts, zeros, iters=12, gpu_verify=False):
    ts = []
    for it in range(iters):
        for r in range(1, n):
            hosts[r].copy_(zeros[:hosts[r].numel()])
        w = B.run_bcast_host(comms, 0, hosts, m, cfg)
        if gpu_verify:
            for r in range(1, n):
                check.copy_(hosts[r])
                assert torch.equal(check, bufs[0])
        else:
            assert all(torch.equal(hosts[r], hosts[0]) for r in range(1, n))
        ts.append(w)
    print(f"{tag}: " + " ".join(f"{t * 1e3:.2f}" for t in ts) + f"  | median {statistics.median(ts[2:]) * 1e3:.3f} ms",
          flush=True)


hosts = [torch.empty(m, dtype=torch.uint8, pin_memory=True) for _ in range(n)]
hosts[0].copy_(bufs[0].cpu())
zeros = torch.zeros(m, dtype=torch.uint8, device=dev)
e2e("fresh", hosts, zeros)
s = torch.cuda.Stream()
for it in range(25):
    with torch.cuda.stream(s):
        for r in range(1, n):
            bufs[r].zero_()
        torch.sum(flush)
    B.bcast_all(comms, bufs, m, "uint8", 0, cfg, streams=[s] * n)
torch.cuda.synchronize()
e2e("after device loop", hosts, zeros)
hosts2 = [torch.empty(m, dtype=torch.uint8, pin_memory=True) for _ in range(n)]
hosts2[0].copy_(bufs[0].cpu())
e2e("new host buffers", hosts2, zeros)
e2e("again", hosts2, zeros)
e2e("gpu verify", hosts2, zeros, gpu_verify=True)
hosts3 = [torch.empty(m, dtype=torch.uint8, pin_memory=True) for _ in range(n)]
hosts3[0].copy_(bufs[0].cpu())
e2e("gpu verify, new buffers", hosts3, zeros, gpu_verify=True)
e2e("cpu verify after", hosts3, zeros)
