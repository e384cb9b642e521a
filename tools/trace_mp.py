#!/usr/bin/env python3
"""Dev tool (torchrun, one process per GPU): bench-shaped broadcast with the
device timeline enabled; each rank prints its kernel time (CUDA events) and
its in-kernel lane span, plus the first/last lane entry relative to ev0."""
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
m = int(os.environ.get("TRACE_BYTES", 1 << 30)); chunk = int(os.environ.get("TRACE_CHUNK", 512 << 10))
comm = B.Comm.connect_torch(world, rank, local, heap_bytes=m + (64 << 20), timeout_s=30)
L = comm.info()["lanes"]
buf = torch.as_tensor(DevicePtr(comm.alloc(m), m), device=dev)
ref = torch.randint(0, 256, (m,), dtype=torch.uint8, device=dev, generator=torch.Generator(device=dev).manual_seed(1))
torch.cuda.synchronize()  # ref is written on the default stream; s reads it
cap = 1024
tr = torch.zeros(L * cap * 4, dtype=torch.int64, device=dev)
cfg = B.AlgorithmConfig(B.Algorithm.chain_pipelined, 0, chunk)
comm.set_protocol(os.environ.get("TRACE_PROTO", "pull"))  # the timeline records the lane executor only
s = torch.cuda.Stream(device=dev)
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
evb = torch.cuda.Event(enable_timing=True)
tstamp = torch.zeros(2, dtype=torch.int64, device=dev)
def chk(tag):
    torch.cuda.synchronize()
    if rank == 0 and not torch.equal(buf, ref):
        bad = int((buf != ref).sum())
        print(f"rank 0 CHECK {tag}: {bad} bad bytes", flush=True)
ITERS = int(os.environ.get("TRACE_ITERS", 5))
ktimes = []
for it in range(ITERS):
    with torch.cuda.stream(s):
        (buf.copy_(ref) if rank == 0 else buf.zero_())
    if it == 0: chk("after copy_")
    with torch.cuda.stream(s):
        tr.zero_()
    if it == 0: chk("after tr.zero_")
    comm.set_trace(tr if it == ITERS - 1 else None, cap)
    s.synchronize(); dist.barrier(device_ids=[local])
    if rank == 0 and not torch.equal(buf, ref):
        print(f"rank 0 iter {it}: root buffer differs BEFORE the broadcast", flush=True)
    with torch.cuda.stream(s):
        torch.cuda._sleep(1_000_000)
    evb.record(s)
    comm.barrier(s)
    ev0.record(s)
    comm.bcast(buf, m, "uint8", 0, cfg, stream=s)
    ev1.record(s)
    ev1.synchronize()
    ktimes.append(ev0.elapsed_time(ev1) * 1e3)
    comm.check(s)
    if not torch.equal(buf, ref):
        bad = (buf != ref).nonzero().flatten()
        print(f"rank {rank} iter {it}: {len(bad)} bad bytes first {int(bad[0])} last {int(bad[-1])} "
              f"chunk {int(bad[0]) // chunk} off {int(bad[0]) % chunk}", flush=True)
        if rank == 0:
            b0 = int(bad[0])
            print("root buf", buf[b0:b0+16].tolist(), "ref", ref[b0:b0+16].tolist(), flush=True)
            # runs of bad bytes
            d = (bad[1:] - bad[:-1])
            brk = (d != 1).nonzero().flatten()
            print("bad runs:", int(len(brk)) + 1, "first run len", int(brk[0]) + 1 if len(brk) else len(bad), flush=True)
        raise SystemExit(1)
life = tr.view(L, cap, 4)[:, cap - 1].cpu()
rec = tr.view(L, cap, 4)[:, :cap - 1].cpu()
act = life[:, 0] > 0
t_in = int(life[:, 0][act].min()); t_in_max = int(life[:, 0][act].max()); t_out = int(life[:, 3][act].max())
land = rec[:, :, 1]; lm = land > 0
msg = (f"rank {rank}: median kernel {statistics.median(ktimes[1:]):.1f}us barrier {evb.elapsed_time(ev0)*1e3:.1f}us kernel(ev0-ev1) {ev0.elapsed_time(ev1)*1e3:.1f}us "
       f"lanes enter span {(t_in_max-t_in)/1e3:.1f}us exit at {(t_out-t_in)/1e3:.1f}us")
if lm.any():
    msg += f" first_land {(int(land[lm].min())-t_in)/1e3:.1f}us last_land {(int(land[lm].max())-t_in)/1e3:.1f}us"
out = [None] * world
dist.all_gather_object(out, msg)
if rank == 0:
    print("\n".join(out))
# cross-rank milestones on the (driver-synchronised) globaltimer
def mn(x): return int(x[x > 0].min()) if (x > 0).any() else 0
def mx(x): return int(x.max())
ms = dict(enter=t_in, enter_last=t_in_max, first_issue=mn(rec[:, :, 0]), first_land=mn(rec[:, :, 1]),
          last_land=mx(rec[:, :, 1]), last_store=mx(rec[:, :, 2]), last_post=mx(rec[:, :, 3]), exit=t_out)
allms = [None] * world
dist.all_gather_object(allms, ms)
if rank == 0:
    base = min(d["enter"] for d in allms)
    for r, d in enumerate(allms):
        print(f"rank {r} (us from first enter): " + " ".join(f"{k}={(v - base) / 1e3:.2f}" if v else f"{k}=-"
                                                            for k, v in d.items()))
npz = os.environ.get("TRACE_NPZ")
if npz:
    import numpy as np
    np.savez_compressed(npz.replace("RANK", str(rank)), rec=tr.view(L, cap, 4).cpu().numpy(),
                        plan=np.array(list(comm.plan(cfg, 0, m).values())), ktimes=np.array(ktimes))
csv_path = os.environ.get("TRACE_CSV")
if csv_path:
    from paper_1707_09414_b200.timeline import chain_rows, write_csv
    plan = comm.plan(cfg, 0, m)
    rows = chain_rows(tr.cpu().numpy(), L, cap, plan, world, 0, rank)
    allrows = [None] * world
    dist.all_gather_object(allrows, rows)
    if rank == 0:
        write_csv([r for part in allrows for r in part], csv_path)
        print("wrote", csv_path, "plan", plan)
dist.barrier(device_ids=[local]); comm.close(); dist.destroy_process_group()
