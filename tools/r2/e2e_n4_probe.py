#!/usr/bin/env python3
"""Dev probe (torchrun, one process per GPU): the N>1 host-buffer broadcast
(bcl_bcast_host) against the same pipeline written out in Python with events
after every piece's H2D, broadcast and D2H, to see where the N=4 e2e time
goes. Prints rank 0's H2D timeline and every receiver's per-piece bcast-done /
D2H-done times (ms from a common start on each rank's stream)."""
import os
import statistics
import time
import torch
import torch.distributed as dist

import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1707_09414_b200 as B  # noqa: E402
from paper_1707_09414_b200.comm import DevicePtr  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
M = 64 << 20
comm = B.Comm.connect_torch(world, rank, local, heap_bytes=3 * M, timeout_s=30)
host = torch.empty(M, dtype=torch.uint8, pin_memory=True)
ref = torch.randint(0, 256, (M,), dtype=torch.uint8, device=dev, generator=torch.Generator(device=dev).manual_seed(1))
scratch = torch.as_tensor(DevicePtr(comm.alloc(M), M), device=dev)
stream, cin, cout = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
zeros = torch.zeros(M, dtype=torch.uint8, device=dev)


def pieces(total, piece=16 << 20):
    out, off, cur = [], 0, min(piece, 1 << 20)
    while off < total:
        if off:
            cur = min(piece, cur * 2)
        out.append((off, min(cur, total - off)))
        off += out[-1][1]
    return out


def reset():
    (host.copy_(ref) if rank == 0 else host.copy_(zeros))
    torch.cuda.synchronize()
    dist.barrier(device_ids=[local])


def lib_path():
    reset()
    t0 = time.perf_counter()
    comm.bcast_host(host, M, "uint8", 0, None, stream=stream)
    stream.synchronize()
    return time.perf_counter() - t0


def py_path():
    reset()
    start = torch.cuda.Event(enable_timing=True)
    marks = []
    t0 = time.perf_counter()
    start.record(stream)
    cin.wait_stream(stream)
    cout.wait_stream(stream)
    for off, ln in pieces(M):
        if rank == 0:
            with torch.cuda.stream(cin):
                scratch[off:off + ln].copy_(host[off:off + ln], non_blocking=True)
            e_in = torch.cuda.Event(enable_timing=True)
            e_in.record(cin)
            stream.wait_event(e_in)
            marks.append(("h2d", ln, e_in))
        comm.bcast(scratch[off:off + ln], ln, "uint8", 0, None, stream=stream)
        e_b = torch.cuda.Event(enable_timing=True)
        e_b.record(stream)
        marks.append(("bcast", ln, e_b))
        if rank != 0:
            cout.wait_event(e_b)
            with torch.cuda.stream(cout):
                host[off:off + ln].copy_(scratch[off:off + ln], non_blocking=True)
            e_o = torch.cuda.Event(enable_timing=True)
            e_o.record(cout)
            marks.append(("d2h", ln, e_o))
    stream.wait_stream(cout)
    stream.synchronize()
    w = time.perf_counter() - t0
    return w, [(k, ln >> 20, round(start.elapsed_time(e), 3)) for k, ln, e in marks]


libs = [lib_path() for _ in range(6)][1:]
pys = [py_path() for _ in range(6)][1:]
ok = torch.equal(host, ref.cpu()) if rank else True
res = [None] * world
dist.all_gather_object(res, (rank, round(statistics.median(libs) * 1e3, 3), round(statistics.median(p[0] for p in pys) * 1e3, 3),
                             pys[-1][1], ok))
if rank == 0:
    for r, lib, py, marks, ok in res:
        print(f"rank {r}: bcast_host {lib} ms, python pipeline {py} ms, ok={ok}")
        print("   ", " ".join(f"{k}{ln}M@{t}" for k, ln, t in marks))
dist.barrier(device_ids=[local])
comm.close()
dist.destroy_process_group()
