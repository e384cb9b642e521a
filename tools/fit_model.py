#!/usr/bin/env python3
"""how well does the reference's analytical model describe
B200? Fit Eq. 5 (chain_pipelined: (ceil(M/C) + n - 2)(t_s + C/B),
models.cpp:75-90) to measured chain latencies, re-run the reference tuner with
the fitted parameters, and compare the reference simulator's per-rank
completion times with a measured device timeline (same trace CSV schema).

  python tools/fit_model.py RAW.csv [MEASURED_TRACE.csv N M CHUNK] > report.txt
"""
import csv
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1707_09414_b200 as B  # noqa: E402

HARNESS = os.path.join(ROOT, "oracle", "_ref", "ref_harness")


def main():
    raw, seen = [], set()
    want = os.environ.get("FIT_PROTO")  # e.g. pull: only the lane executor's measurements
    for r in csv.DictReader(open(sys.argv[1])):  # first measurement of a point = the default protocol
        if want is not None and r.get("protocol", "auto") != want:
            continue
        if want is None and r.get("protocol", "auto") != "auto":
            continue
        key = (r["algorithm"], r["radix"], r["chunk_bytes"], r["n"], r["bytes"])
        if key not in seen:
            seen.add(key)
            raw.append(r)
    chain = [r for r in raw if r["algorithm"] == "chain_pipelined" and int(r["bytes"]) >= 1 << 20]
    rows, y = [], []
    for r in chain:
        m, c, n = int(r["bytes"]), int(r["chunk_bytes"]), int(r["n"])
        k = -(-m // c) + n - 2
        rows.append([1.0, k, k * c])
        y.append(float(r["seconds"]))
    A, y = np.array(rows, dtype=float), np.array(y)

    def fit(cols, label):
        # relative-error least squares: every size counts, not just the largest
        coef, *_ = np.linalg.lstsq(A[:, cols] / y[:, None], np.ones_like(y), rcond=None)
        coef = np.maximum(coef, 1e-12)
        pred = A[:, cols] @ coef
        rel = np.abs(pred - y) / y
        print(f"{label}: median rel. error {np.median(rel):.1%}, max {rel.max():.1%}")
        for i in np.argsort(-rel)[:4]:
            r = chain[i]
            print(f"    n={r['n']} M={r['bytes']} C={r['chunk_bytes']}: measured {y[i]*1e6:.1f} us, "
                  f"model {pred[i]*1e6:.1f} us")
        return coef

    print(f"least-squares fits over {len(y)} measured chain_pipelined points (M >= 1 MiB)")
    ts, inv_b = (float(v) for v in fit([1, 2], "Eq. 5 as the reference states it, (K+n-2)(t_s + C/B)"))
    print(f"  t_s = {ts * 1e6:.3f} us, B = {1 / inv_b / 1e9:.1f} GB/s")
    a0, ts2, inv_b2 = (float(v) for v in fit([0, 1, 2], "Eq. 5 + a per-call constant a0"))
    print(f"  a0 = {a0 * 1e6:.2f} us, t_s = {ts2 * 1e6:.3f} us, B = {1 / inv_b2 / 1e9:.1f} GB/s")
    # tuner with the fitted analytical oracle vs the measured table
    sizes = [4 << i for i in range(29)]
    cands = [B.AlgorithmConfig.of("knomial", 2), B.AlgorithmConfig.of("scatter_ring_allgather"),
             B.AlgorithmConfig.of("chain_pipelined"), B.AlgorithmConfig.of("direct")]
    chunks = [65536 << i for i in range(7)]
    ns = sorted({int(r["n"]) for r in raw})
    t = B.tune(ns, sizes, cands, chunks, startup_s=max(ts, 1e-9), link_Bps=1 / inv_b)
    print("\nanalytical table with the fitted parameters:")
    print(t.text())
    print("measured (builtin) table:")
    print(B.builtin_table().text())
    if len(sys.argv) > 5 and os.path.exists(HARNESS):
        trace, n, m, c = sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
        out = subprocess.run([HARNESS, "simulate", "chain_pipelined", str(n), "0", str(m), str(c), "0",
                              repr(max(ts2, 1e-9)), repr(1 / inv_b2), "/tmp/sim_trace.csv"],
                             capture_output=True, text=True, check=True).stdout
        sim = {int(l.split()[1]): float(l.split()[2]) + a0 for l in out.splitlines()}
        meas = {}
        for r in csv.DictReader(open(trace)):
            meas[int(r["rank"])] = max(meas.get(int(r["rank"]), 0.0), float(r["end_s"]))
        print(f"per-rank completion, chain n={n} M={m} C={c}: reference simulator (fitted, + a0) vs measured B200")
        for rk in range(n):
            print(f"  rank {rk}: simulated {sim.get(rk, 0) * 1e6:9.1f} us   measured {meas.get(rk, 0) * 1e6:9.1f} us")


if __name__ == "__main__":
    main()
