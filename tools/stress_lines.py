#!/usr/bin/env python3
"""Robustness run for the line protocols across GPUs (one process drives
every visible GPU): ITERS back-to-back broadcasts with random sizes
(1 B - 128 MiB, log-uniform), rotating roots, fresh payloads, alternating
LL128 / LL / auto; every receiver checked byte-exact before the next call
reuses the landing halves. Prints one summary line."""
import math, os, random, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1707_09414_b200 as B
iters = int(os.environ.get("ITERS", 400))
devs = list(range(torch.cuda.device_count()))
n = len(devs)
comms = B.Comm.local(devs, timeout_s=20)
cap = 128 << 20
bufs = [torch.empty(cap, dtype=torch.uint8, device=f"cuda:{d}") for d in devs]
rng = random.Random(int(os.environ.get("SEED", 7)))
cfg = B.AlgorithmConfig(B.Algorithm.chain_pipelined, 0, 262144)
counts = {"ll128": 0, "ll": 0, "auto": 0}
t0 = time.time()
for it in range(iters):
    proto = ("ll128", "ll", "auto")[it % 3]
    hi = (8 << 20) if proto == "ll" else cap
    m = max(1, int(math.exp(rng.uniform(0, math.log(hi)))))
    root = rng.randrange(n)
    for c in comms:
        c.set_protocol(proto)
    src = torch.randint(0, 256, (m,), dtype=torch.uint8, device=f"cuda:{devs[root]}")
    for r in range(n):
        (bufs[r][:m].copy_(src) if r == root else bufs[r][:m].fill_((it * 37 + r) & 0xFF))
    for d in devs:
        torch.cuda.synchronize(d)
    B.run_bcast(comms, root, [b[:m] for b in bufs], m, cfg)
    for r in range(n):
        if not torch.equal(bufs[r][:m].cpu(), src.cpu()):
            bad = int((bufs[r][:m].cpu() != src.cpu()).sum())
            raise SystemExit(f"MISMATCH it={it} proto={proto} m={m} root={root} rank={r} bad_bytes={bad}")
    counts[proto] += 1
print(f"stress ok: {iters} broadcasts on {n} GPUs in {time.time() - t0:.0f} s, per protocol {counts}")
