#!/usr/bin/env python3
"""Dev probe (torchrun, one process per GPU): the N>1 host-buffer shape --
rank 0 H2D of M, every other rank D2H of M, all at once -- with the pinned
buffers allocated (a) wherever the process runs, (b) after pinning the process
to its GPU's local CPUs (/sys/bus/pci/devices/<bus id>/local_cpulist), so the
pages sit on the GPU's NUMA node. Per-rank DMA time (events), median of 7."""
import os
import statistics
import sys
import torch
import torch.distributed as dist

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
M = 64 << 20


def local_cpus():
    bus = torch.cuda.get_device_properties(local).pci_bus_id if hasattr(torch.cuda.get_device_properties(local), "pci_bus_id") else None
    if bus is None:
        import subprocess
        out = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader", "-i", str(local)],
                             capture_output=True, text=True).stdout.strip()
        bus = out
    bus = bus.lower()
    if bus.startswith("0000") and len(bus.split(":")[0]) == 8:
        bus = bus[4:]
    for cand in (bus, "0000" + bus[4:] if bus.startswith("0000") else "0000:" + bus.split(":", 1)[-1]):
        p = f"/sys/bus/pci/devices/{cand}/local_cpulist"
        if os.path.exists(p):
            txt = open(p).read().strip()
            cpus = set()
            for part in txt.split(","):
                a, _, b = part.partition("-")
                cpus.update(range(int(a), int(b or a) + 1))
            return cpus, p, open(f"/sys/bus/pci/devices/{cand}/numa_node").read().strip()
    return None, bus, "?"


def measure(tag):
    host = torch.empty(M, dtype=torch.uint8, pin_memory=True)
    host.fill_(1)
    d = torch.empty(M, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream(device=dev)
    ts = []
    for it in range(8):
        torch.cuda.synchronize()
        dist.barrier(device_ids=[local])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        with torch.cuda.stream(s):
            (d.copy_(host, non_blocking=True) if rank == 0 else host.copy_(d, non_blocking=True))
        e1.record(s)
        e1.synchronize()
        if it:
            ts.append(e0.elapsed_time(e1))
    t = statistics.median(ts)
    all_t = [None] * world
    dist.all_gather_object(all_t, (rank, round(t, 3), os.sched_getaffinity(0).__len__()))
    if rank == 0:
        print(f"{tag}: " + ", ".join(f"rank {r} {'H2D' if r == 0 else 'D2H'} {x} ms ({M / x / 1e6:.1f} GB/s, {c} cpus)"
                                     for r, x, c in all_t), flush=True)


measure("unpinned process")
cpus, where, node = local_cpus()
info = [None] * world
dist.all_gather_object(info, (rank, where, node, len(cpus) if cpus else 0))
if rank == 0:
    print("GPU-local CPUs:", info, flush=True)
if cpus:
    os.sched_setaffinity(0, cpus)
measure("process pinned to its GPU's NUMA node")
dist.barrier(device_ids=[local])
dist.destroy_process_group()
