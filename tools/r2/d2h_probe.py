#!/usr/bin/env python3
"""Dev probe (torchrun, one process per GPU): concurrent host DMA of the N>1
e2e shape, each rank's span from a common barrier to its last copy: (a) the
receivers' D2H of 64 MiB in 16 MiB pieces, (b) the same with rank 0's H2D of
64 MiB, (c) (b) while every GPU runs a spinning kernel on another stream,
(d) (b) while every GPU runs the broadcast's LL128 chain kernels (piece-sized
broadcasts issued on another stream, waiting on the root)."""
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
M = 64 << 20
P = 16 << 20
comm = B.Comm.connect_torch(world, rank, local, heap_bytes=2 * M, timeout_s=30)
scr = torch.as_tensor(DevicePtr(comm.alloc(M), M), device=dev)
d = torch.empty(M, dtype=torch.uint8, device=dev)
host = torch.empty(M, dtype=torch.uint8, pin_memory=True)
s_copy, s_kern = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)


def once(h2d, side):
    torch.cuda.synchronize()
    dist.barrier(device_ids=[local])
    t0 = time.perf_counter()
    if side == "spin":
        with torch.cuda.stream(s_kern):
            torch.cuda._sleep(2_000_000)
    if side == "bcast":
        for k in range(M // P):
            comm.bcast(scr[k * P:(k + 1) * P], P, "uint8", 0, None, stream=s_kern)
    with torch.cuda.stream(s_copy):
        if rank == 0:
            if h2d:
                d.copy_(host, non_blocking=True)
        else:
            for k in range(M // P):
                host[k * P:(k + 1) * P].copy_(d[k * P:(k + 1) * P], non_blocking=True)
    s_copy.synchronize()
    t = time.perf_counter() - t0
    s_kern.synchronize()
    return t


out = []
for tag, h2d, side in (("D2H only", False, None), ("D2H + root H2D", True, None), ("+ spinning kernel", True, "spin"),
                       ("+ LL128 chain broadcasts", True, "bcast")):
    ts = [once(h2d, side) for _ in range(6)][1:]
    res = [None] * world
    dist.all_gather_object(res, round(statistics.median(ts) * 1e3, 3))
    if rank == 0:
        print(f"{tag}: per-rank copy span ms {res}", flush=True)
dist.barrier(device_ids=[local])
comm.close()
dist.destroy_process_group()
