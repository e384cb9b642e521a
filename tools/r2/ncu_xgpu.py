#!/usr/bin/env python3
"""ncu target for the cross-GPU kernels (dev tool): ONE process drives two
GPUs (root rank 0 on cuda:0, receiver rank 1 on cuda:1) and runs ONE
broadcast, so `ncu --devices 1` (or 0) can profile a real NVLink kernel.

ncu serialises kernel launches: the root's kernel runs alone first. On the
pull path it publishes its flags and mailboxes, then waits for the receiver's
acks until its device timeout (--timeout, default 3 s) fires; the receiver's
kernel then runs with every flag already set and pulls the whole message over
NVLink (every ncu replay repeats exactly that). LL128 up to ~54 MB never waits
at the root (each warp writes fewer groups than its ring depth), so both
kernels complete. NVLS below the 64 MiB ring never waits at the root either
(the root's multicast stores land in every GPU's ring copy; the receiver then
copies its copy out). Without ncu both kernels run concurrently and the call
succeeds; the receiver's buffer is verified either way.

`direct128` / `direct_ll`: the `direct` schedule on LL128 direct lines / on
16-byte LL lines (ll128_direct_min=0), BYTES <= 2 MiB; the root never waits
on a first call, so both kernels complete under ncu too.

  python tools/r2/ncu_xgpu.py pull|ll128|pull_vec|nvls|direct128|direct_ll BYTES [--timeout S]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
import paper_1707_09414_b200 as B  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["pull", "ll128", "pull_vec", "nvls", "direct128", "direct_ll"])
    ap.add_argument("bytes", type=int)
    ap.add_argument("--chunk", type=int, default=65536)
    ap.add_argument("--timeout", type=float, default=3.0)
    args = ap.parse_args()
    opts = {"stage_bytes": 0} if args.mode == "pull_vec" else {"ll128_direct_min": 0} if args.mode == "direct_ll" else {}
    comms = B.Comm.local([0, 1], timeout_s=args.timeout, **opts)
    for c in comms:
        c.set_protocol({"ll128": "ll128", "nvls": "nvls"}.get(args.mode, "pull"))
    m = args.bytes
    bufs = [torch.zeros(m, dtype=torch.uint8, device=f"cuda:{d}") for d in (0, 1)]
    bufs[0].copy_(torch.randint(0, 256, (m,), dtype=torch.uint8, device="cuda:0",
                                generator=torch.Generator(device="cuda:0").manual_seed(3)))
    torch.cuda.synchronize(0)
    cfg = B.AlgorithmConfig(B.Algorithm.chain_pipelined, 0, args.chunk)
    if args.mode.startswith("direct"):
        for c in comms:
            c.set_protocol("auto")
        cfg = B.AlgorithmConfig(B.Algorithm.direct, 0, 0)
        print("path:", comms[0].path(m, cfg))
    B.bcast_all(comms, bufs, m, "uint8", 0, cfg)
    status = []
    for r, c in enumerate(comms):
        try:
            c.check()
            status.append("ok")
        except B.BclError as e:  # the root's ack wait under ncu serialisation
            status.append(type(e).__name__)
    ok = torch.equal(bufs[1].cpu(), bufs[0].cpu())
    print(f"{args.mode} M={m}: ranks {status}, receiver bit-exact={ok}")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
