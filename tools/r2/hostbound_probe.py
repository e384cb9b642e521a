#!/usr/bin/env python3
"""Dev probe (torchrun, one process per GPU): are small back-to-back
broadcasts host-bound? 50 calls of S bytes eager (Python -> C-ABI per call)
against the same 50 calls captured in a CUDA graph and replayed (no host work
per call), device time between events, max over ranks; plus the host-side
enqueue time per eager call."""
import os
import statistics
import sys
import time
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1707_09414_b200 as B  # noqa: E402
from paper_1707_09414_b200.comm import DevicePtr  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
comm = B.Comm.connect_torch(world, rank, local, heap_bytes=64 << 20, timeout_s=30)
buf = torch.as_tensor(DevicePtr(comm.alloc(4 << 20), 4 << 20), device=dev)
s = torch.cuda.Stream(device=dev)
CALLS = 50


def maxr(x):
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


for size in (8, 4096, 65536, 1 << 20):
    cfg = comm.choose(size)
    eager, host = [], []
    for rep in range(6):
        torch.cuda.synchronize()
        dist.barrier(device_ids=[local])
        with torch.cuda.stream(s):
            torch.cuda._sleep(1_000_000)
        comm.barrier(s)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        h0 = time.perf_counter()
        for _ in range(CALLS):
            comm.bcast(buf, size, "uint8", 0, cfg, stream=s)
        h1 = time.perf_counter()
        e1.record(s)
        e1.synchronize()
        if rep:
            eager.append(e0.elapsed_time(e1) * 1e3 / CALLS)
            host.append((h1 - h0) * 1e6 / CALLS)
    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        for _ in range(CALLS):
            comm.bcast(buf, size, "uint8", 0, cfg, stream=s)
    torch.cuda.synchronize()
    graph = []
    for rep in range(6):
        torch.cuda.synchronize()
        dist.barrier(device_ids=[local])
        with torch.cuda.stream(s):
            torch.cuda._sleep(1_000_000)
        comm.barrier(s)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        with torch.cuda.stream(s):
            g.replay()
        e1.record(s)
        e1.synchronize()
        if rep:
            graph.append(e0.elapsed_time(e1) * 1e3 / CALLS)
    del g
    r = (maxr(statistics.median(eager)), maxr(statistics.median(graph)), maxr(statistics.median(host)))
    if rank == 0:
        print(f"N={world} {size} B [{comm.path(size, cfg)}]: eager {r[0]:.2f} us/call, graph replay {r[1]:.2f} us/call, "
              f"host enqueue {r[2]:.2f} us/call", flush=True)
comm.check(s)
dist.barrier(device_ids=[local])
comm.close()
dist.destroy_process_group()
