#!/usr/bin/env python3
"""Dev A/B (torchrun, one process per GPU): device time of the pipelined
chain per transport variant and size (GPU gate, device barrier, CUDA events,
median of K, max over ranks). VARIANTS: ';'-separated "protocol[:k=v,...]";
ALGO: the schedule (chain_pipelined, direct, ..., or "table": the tuned
choice); B2B: calls per timed region (back to back, one event pair)."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch, torch.distributed as dist
import paper_1707_09414_b200 as B
from paper_1707_09414_b200.comm import DevicePtr
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
sizes = [int(x) for x in os.environ.get("SIZES", "8388608,67108864,268435456,1073741824").split(",")]
chunk = int(os.environ.get("CHUNK", 65536))
K = int(os.environ.get("ITERS", 10))
variants = os.environ.get("VARIANTS", "ll128;ll128:ll128_coop=0;pull;push").split(";")
B2B = int(os.environ.get("B2B", 1))
ALGO = os.environ.get("ALGO", "chain_pipelined")
mx = max(sizes)
s = torch.cuda.Stream(device=dev)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for v in variants:
    proto, _, opts = v.partition(":")
    options = dict(kv.split("=") for kv in opts.split(",") if kv)
    comm = B.Comm.connect_torch(world, rank, local, heap_bytes=mx + (16 << 20), timeout_s=30, **options)
    comm.set_protocol(proto)
    buf = torch.as_tensor(DevicePtr(comm.alloc(mx), mx), device=dev)
    ref = torch.randint(0, 256, (mx,), dtype=torch.uint8, device=dev, generator=torch.Generator(device=dev).manual_seed(5))
    torch.cuda.synchronize()
    res = []
    for m in sizes:
        cfg = None if ALGO == "table" else B.AlgorithmConfig(
            B.Algorithm[ALGO], 2 if ALGO == "knomial" else 0, chunk if ALGO == "chain_pipelined" else 0)
        ts = []
        for it in range(3 + K):
            with torch.cuda.stream(s):
                (buf[:m].copy_(ref[:m]) if rank == 0 else buf[:m].zero_())
                torch.cuda._sleep(1_000_000)
            comm.barrier(s)
            e0.record(s)
            for _ in range(B2B):
                comm.bcast(buf, m, "uint8", 0, cfg, stream=s)
            e1.record(s)
            e1.synchronize()
            if it >= 3:
                ts.append(e0.elapsed_time(e1) * 1e-3 / B2B)
        ok = torch.equal(buf[:m], ref[:m])
        t = torch.tensor(ts, dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        okt = torch.tensor([1.0 if ok else 0.0], device=dev)
        dist.all_reduce(okt, op=dist.ReduceOp.MIN)
        med = statistics.median(t.cpu().tolist())
        res.append(f"{m >> 10}KiB {med * 1e6:.1f}us {m / med / 1e9:.0f}GB/s{'' if okt.item() else ' MISMATCH'}")
    if rank == 0:
        print(f"N={world} {v} {ALGO} b2b={B2B} [{comm.path(sizes[-1], cfg)}]: " + " | ".join(res), flush=True)
    comm.close()
dist.barrier(device_ids=[local])
dist.destroy_process_group()
