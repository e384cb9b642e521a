#!/usr/bin/env python3
"""Dev tool (torchrun, one process per GPU): chain_pipelined device latency
under a grid of GroupOptions environment settings (each setting builds a
fresh communicator), max over ranks, median over iterations.

  SWEEP='BCL_WINDOW_BYTES=1048576;BCL_MAX_CTAS=74' SIZES=67108864 CHUNKS=65536,524288 \
    torchrun --nproc-per-node 4 tools/sweep_opts.py
Settings are separated by ';', variables within a setting by ','."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
import paper_1707_09414_b200 as B
from paper_1707_09414_b200.comm import DevicePtr

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
sizes = [int(x) for x in os.environ.get("SIZES", str(64 << 20)).split(",")]
chunks = [int(x) for x in os.environ.get("CHUNKS", "65536,524288").split(",")]
settings = [""] + [s for s in os.environ.get("SWEEP", "").split(";") if s]
iters = int(os.environ.get("ITERS", 15))
proto = os.environ.get("PROTO", "auto")
M = max(sizes)
for setting in settings:
    saved = {}
    for kv in [x for x in setting.split(",") if x]:
        k, v = kv.split("=")
        saved[k] = os.environ.get(k)
        os.environ[k] = v
    comm = B.Comm.connect_torch(world, rank, local, heap_bytes=M + (64 << 20), timeout_s=30)
    comm.set_protocol(proto)
    buf = torch.as_tensor(DevicePtr(comm.alloc(M), M), device=dev)
    buf.fill_(7 if rank == 0 else 0)
    s = torch.cuda.Stream(device=dev)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    line = []
    for m in sizes:
        for c in chunks:
            algo = B.Algorithm[os.environ.get("ALGO", "chain_pipelined")]
            cfg = B.AlgorithmConfig(algo, 0, c if algo == B.Algorithm.chain_pipelined else 0)
            ts = []
            for it in range(3 + iters):
                with torch.cuda.stream(s):
                    torch.cuda._sleep(int(os.environ.get("GATE", 400_000)))
                comm.barrier(s)
                ev0.record(s)
                comm.bcast(buf, m, "uint8", 0, cfg, stream=s)
                ev1.record(s)
                ev1.synchronize()
                if it >= 3:
                    ts.append(ev0.elapsed_time(ev1) * 1e3)
            t = torch.tensor(ts, dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            med = statistics.median(t.cpu().tolist())
            line.append(f"M={m} C={c}: {med:.1f}us ({m / med / 1e3:.0f} GB/s)")
    comm.check(s)
    ok = bool((buf[:M] == 7).all())
    if rank == 0:
        print(f"[{setting or 'default'}] lanes={comm.info()['lanes']} ok={ok} | " + " | ".join(line), flush=True)
    comm.close()
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k)
        else:
            os.environ[k] = v
dist.destroy_process_group()
