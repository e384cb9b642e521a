#!/usr/bin/env python3
"""Re-derive the tuning table on B200 from MEASURED latencies (the paper's
collective tuning framework, with a Measured oracle).

  torchrun --nproc-per-node N tools/tune_b200.py --out tables/b200_measured_nN.csv

Runs the reference tuner algorithm (bcl::tune: argmin per swept size,
geometric-mean range bounds, merged ranges, tie-breaks of tuner.cpp:84-92)
with cost(config, n, M) = median over iterations of the max-over-ranks device
latency of our broadcast (GPU-gated, device-barrier-aligned, CUDA events).
Every rank evaluates the same candidate sequence, so each cost call is a
collective measurement."""
import argparse
import math
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
import paper_1707_09414_b200 as B  # noqa: E402
from paper_1707_09414_b200.comm import DevicePtr  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", required=True)
ap.add_argument("--min", "--min-bytes", dest="min", type=int, default=4)
ap.add_argument("--max", "--max-bytes", dest="max", type=int, default=1 << 30)  # (--max-bytes under torchrun)
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--chunks", default="65536,131072,262144,524288,1048576,2097152,4194304")
ap.add_argument("--cands", default="direct,knomial,scatter_ring_allgather,chain_pipelined")
ap.add_argument("--raw", default="", help="also write every measurement (config, n, bytes, seconds) here")
ap.add_argument("--b2b", type=int, default=1,
                help="cost = mean of this many calls issued back to back (what a training step issues; resolves "
                     "differences below the ~2 us event tick); 1 = single gated calls")
a = ap.parse_args()

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
comm = B.Comm.connect_torch(world, rank, local, heap_bytes=a.max + (64 << 20), timeout_s=30)
buf = torch.as_tensor(DevicePtr(comm.alloc(a.max), a.max), device=dev)
buf.fill_(7 if rank == 0 else 0)
stream = torch.cuda.Stream(device=dev)
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n_eval = [0]
raw = []
proto_now = ["auto"]


def set_proto(p):
    proto_now[0] = p
    comm.set_protocol(p)


def quantize(t):
    """2 significant digits: costs closer than the timer noise tie, and ties
    fall to the reference's tie-break order (tuner.cpp:84-92)."""
    if t <= 0:
        return t
    e = math.floor(math.log10(t)) - 1
    return round(t / 10 ** e) * 10 ** e


def cost(cfg, n, m):
    n_eval[0] += 1
    times = []
    iters = a.iters * 4 if m <= (1 << 20) else a.iters
    for it in range(2 + iters):
        with torch.cuda.stream(stream):
            torch.cuda._sleep(400_000)
        comm.barrier(stream)
        ev0.record(stream)
        try:
            for _ in range(a.b2b if m <= (16 << 20) else 1):
                comm.bcast(buf, m, "uint8", 0, cfg, stream=stream)
        except Exception as e:
            raise RuntimeError(f"bcast {cfg} M={m} protocol={proto_now[0]} failed: {e}") from e
        ev1.record(stream)
        ev1.synchronize()
        if it >= 2:
            times.append(ev0.elapsed_time(ev1) * 1e-3 / (a.b2b if m <= (16 << 20) else 1))
    t = torch.tensor(times, dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    med = float(statistics.median(t.cpu().tolist()))
    raw.append((cfg.algorithm.name, cfg.radix_k, cfg.chunk_bytes, n, m, med, proto_now[0]))
    return quantize(med)


def raw_cost(cfg, n, m):
    """Unquantized median: transport rules compare protocols of one schedule,
    where 2-significant-digit ties (10 us steps above 100 us) would hide
    real differences."""
    cost(cfg, n, m)
    return raw[-1][5]


sizes = []
s = a.min
while s <= a.max:
    sizes.append(s)
    s *= 2
cands = []
for name in a.cands.split(","):
    cands.append(B.AlgorithmConfig.of(name, radix_k=2 if "knomial" in name else 0))
chunks = [int(x) for x in a.chunks.split(",")]
t0 = time.time()
table = B.tune_measured([world], sizes, cands, chunks, cost,
                        provenance=f"B200 x{world}, NVLink (LL128 lines, P2P pulls or pushes per rule), median of {a.iters}-{4 * a.iters} "
                                   f"device-timed runs (max over ranks, 2 significant digits"
                                   f"{f'; mean of {a.b2b} back-to-back calls up to 16 MiB' if a.b2b > 1 else ''}), "
                                   f"{time.strftime('%Y-%m-%d')}")
comm.check(stream)

# Transport protocol for the pipelined chain: measure pull vs push at every
# swept size >= 16 MiB where the table picks the chain; push wins from the
# smallest size after which it always wins ("# bcl-push-from" rule).
push_from = None
if world >= 3:
    wins = []
    for m in [x for x in sizes if x >= (16 << 20)]:
        cfg = table.select(world, m)
        if cfg.algorithm != B.Algorithm.chain_pipelined:
            wins.append((m, False))
            continue
        set_proto("pull")
        t_pull = raw_cost(cfg, world, m)
        set_proto("push")
        t_push = raw_cost(cfg, world, m)
        set_proto("auto")
        wins.append((m, t_push < t_pull))
        if rank == 0:
            print(f"protocol {m}: pull {t_pull * 1e6:.1f} us push {t_push * 1e6:.1f} us")
    for i, (m, w) in enumerate(wins):
        if w and all(x for _, x in wins[i:]):
            push_from = m
            break
    comm.check(stream)

# Line protocol for the chain: LL128 (cross-GPU, up to the landing-area cap)
# against the lane executor (pull, or push past the push-from size) at every
# swept chain size >= 1 MiB. LL128 is used up to the geometric mean of the
# last size where it wins and the first where it loses ("# bcl-ll128-upto").
ll128_upto = None
ll128_cap = comm.protocol_caps()["ll128"]
if ll128_cap:
    last_win = None
    for m in [x for x in sizes if (1 << 20) <= x <= ll128_cap]:
        cfg = table.select(world, m)
        if cfg.algorithm != B.Algorithm.chain_pipelined:
            continue
        set_proto("ll128")
        t_ll = raw_cost(cfg, world, m)
        set_proto("push" if push_from is not None and m >= push_from else "pull")
        t_lane = raw_cost(cfg, world, m)
        set_proto("auto")
        if rank == 0:
            print(f"line protocol {m}: ll128 {t_ll * 1e6:.1f} us lane executor {t_lane * 1e6:.1f} us")
        if t_ll <= t_lane:
            last_win = m
        else:
            ll128_upto = int(math.sqrt(last_win * m)) if last_win else 0
            break
    if ll128_upto is None:
        ll128_upto = ll128_cap
    comm.check(stream)
text = table.text()
extra = []
if push_from is not None:
    extra.append(f"# bcl-push-from: n={world} bytes={push_from}")
if ll128_upto is not None:
    extra.append(f"# bcl-ll128-upto: n={world} bytes={ll128_upto}")
if extra:
    lines = text.splitlines()
    lines[1:1] = extra
    text = "\n".join(lines) + "\n"
    table = B.load_table_text(text)
if rank == 0:
    os.makedirs(os.path.dirname(os.path.abspath(a.out)), exist_ok=True)
    B.save_table(table, a.out)
    if a.raw:
        with open(a.raw, "w") as f:
            f.write("algorithm,radix,chunk_bytes,n,bytes,seconds,protocol\n")
            for r in raw:
                f.write(",".join(map(str, r)) + "\n")
    print(f"wrote {a.out}: {len(table.entries)} entries from {n_eval[0]} measurements in {time.time() - t0:.1f}s")
    print(table.text())
dist.barrier(device_ids=[local])
comm.close()
dist.destroy_process_group()
