#!/usr/bin/env python3
"""The reference CPU broadcast swept over sizes and rank counts on this host
(BASELINE.md §3): the unmodified bcastlab library (oracle/_ref/ref_harness,
osu method: zeroed receivers, barrier, time, verify, max over rank threads),
chain_pipelined with C = min(M, 512 KiB), root 0, inproc transport (and the
socket transport with --socket). One JSON object on stdout with the host's
core count and CPU model.

  python tools/cpu_sweep.py [--ranks 2,4,8] [--max 1073741824] [--socket]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import host_cpu  # noqa: E402

HARNESS = os.path.join(ROOT, "oracle", "_ref", "ref_harness")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", default="2,4,8")
    ap.add_argument("--max", type=int, default=1 << 30)
    ap.add_argument("--socket", action="store_true")
    ap.add_argument("--budget-s", type=float, default=4.0, help="approximate CPU seconds per point")
    args = ap.parse_args()
    if not os.path.exists(HARNESS):
        raise SystemExit(f"{HARNESS} missing: build it with make -C oracle on a host with /root/reference")
    out = {"host": host_cpu(), "algorithm": "chain_pipelined", "chunk": "min(M, 524288)", "root": 0,
           "method": "osu (bcastlab bench): warm-up, zeroed receivers, barrier, verify, max over rank threads",
           "points": []}
    for transport in (["inproc", "socket"] if args.socket else ["inproc"]):
        for n in [int(x) for x in args.ranks.split(",")]:
            size = 4
            while size <= args.max:
                # iterations: ~budget at an assumed ~1 GB/s, between 3 and 20
                iters = int(max(3, min(20, args.budget_s * 1e9 / max(size * n, 1))))
                warm = 1 if size >= (64 << 20) else 2
                chunk = min(size, 512 << 10)
                r = subprocess.run([HARNESS, "bench", "chain_pipelined", str(n), "0", str(size), str(chunk), "0",
                                    str(warm), str(iters), transport, "1"], capture_output=True, text=True,
                                   check=True, timeout=600)
                j = json.loads(r.stdout)
                out["points"].append({"transport": transport, "n": n, "bytes": size, "iters": iters,
                                      "median_us": j["median_us"], "min_us": j["min_us"], "max_us": j.get("max_us"),
                                      "algbw_gbs": round(size / (j["median_us"] * 1e-6) / 1e9, 4),
                                      "ok": j["ok"]})
                print(f"{transport} n={n} M={size}: median {j['median_us']:.1f} us", file=sys.stderr, flush=True)
                size *= 4 if size < (1 << 20) else 2
    print(json.dumps(out))


if __name__ == "__main__":
    main()
