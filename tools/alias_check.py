#!/usr/bin/env python3
"""Dev tool: do the per-process symmetric heaps alias? Each rank fills its own
heap buffer with its rank id, then checks it after the others wrote theirs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
import paper_1707_09414_b200 as B
from paper_1707_09414_b200.comm import DevicePtr
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("gloo")
m = int(os.environ.get("M", 1 << 30))
comm = B.Comm.connect_torch(world, rank, rank, heap_bytes=m + (64 << 20), timeout_s=30)
p = comm.alloc(m)
buf = torch.as_tensor(DevicePtr(p, m), device=dev)
print(f"rank {rank}: heap ptr {p:#x} tensor ptr {buf.data_ptr():#x} device {buf.device}", flush=True)
for step in range(world):
    if step == rank:
        buf.fill_(rank + 1)
        torch.cuda.synchronize()
    dist.barrier()
torch.cuda.synchronize()
bad = int((buf != rank + 1).sum())
u = torch.unique(buf).tolist()
print(f"rank {rank}: bad={bad} values={u[:8]}", flush=True)
ref = torch.randint(0, 256, (m,), dtype=torch.uint8, device=dev)
buf.copy_(ref); torch.cuda.synchronize()
print(f"rank {rank}: copy ok={torch.equal(buf, ref)}", flush=True)
x = torch.empty(m, dtype=torch.uint8, device=dev); x.copy_(ref); torch.cuda.synchronize()
print(f"rank {rank}: torch-alloc copy ok={torch.equal(x, ref)}", flush=True)
dist.barrier(); comm.close(); dist.destroy_process_group()
