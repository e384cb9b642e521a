#!/usr/bin/env python3
"""Dev tool: timeline of the TMA (bulk) chain path across real GPUs.
Per pull record: [0] flag seen, [1] load landed, [2] store issued, [3] published."""
import argparse, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1707_09414_b200 as B
ap = argparse.ArgumentParser()
ap.add_argument("--devices", default="0,1,2,3")
ap.add_argument("--bytes", type=int, default=1 << 30)
ap.add_argument("--chunk", type=int, default=512 << 10)
a = ap.parse_args()
devices = [int(x) for x in a.devices.split(",")]
n, m = len(devices), a.bytes
comms = B.Comm.local(devices, timeout_s=20)
L = comms[0].info()["lanes"]
cfg = B.AlgorithmConfig(B.Algorithm.chain_pipelined, 0, a.chunk)
bufs = [torch.zeros(m, dtype=torch.uint8, device=f"cuda:{d}") for d in devices]
bufs[0].random_(0, 256)
cap = 1024
tr = [torch.zeros(L * cap * 4, dtype=torch.int64, device=f"cuda:{d}") for d in devices]
for it in range(4):
    for r in range(n):
        tr[r].zero_()
        comms[r].set_trace(tr[r] if it == 3 else None, cap)
    for d in devices: torch.cuda.synchronize(d)
    B.bcast_all(comms, bufs, m, "uint8", 0, cfg)
    for d in devices: torch.cuda.synchronize(d)
for r in range(1, n):
    rec = tr[r].view(L, cap, 4)[:, :cap - 1].cpu()
    life = tr[r].view(L, cap, 4)[:, cap - 1].cpu()
    m_ = rec[:, :, 1] > 0
    t0 = int(life[:, 0][life[:, 0] > 0].min())
    f, ld, si, pb = (rec[:, :, i] for i in range(4))
    lat = (ld - f)[m_].double()  # flag seen -> data landed (load latency incl. queueing)
    pv = pb[m_ & (pb > 0)]
    print(f"rank {r}: pulls={int(m_.sum())} load_latency mean={lat.mean()/1e3:.2f}us p50={lat.median()/1e3:.2f} "
          f"first_land={(int(ld[m_].min())-t0)/1e3:.1f}us last_land={(int(ld[m_].max())-t0)/1e3:.1f}us "
          f"last_pub={(int(pv.max())-t0)/1e3 if len(pv) else -1:.1f}us")
    # per-lane gaps: time between consecutive lands of the same lane
    gaps = (ld[:, 1:] - ld[:, :-1])[m_[:, 1:] & m_[:, :-1]].double()
    print(f"          land-to-land per lane mean={gaps.mean()/1e3:.2f}us p50={gaps.median()/1e3:.2f}us p90={gaps.quantile(0.9)/1e3:.2f}us")
    # how far behind upstream: flag seen vs previous land
    pref = (f[:, 1:] < ld[:, :-1]) & m_[:, 1:]
    print(f"          prefetched (flag seen before previous landed): {float(pref.sum())/max(1,int(m_[:,1:].sum())):.2f}")
