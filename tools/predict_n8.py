#!/usr/bin/env python3
"""Predicted n = 8 tuning tables (no 8-GPU box is available: gpurun grants at
most 4 GPUs). Two predictions, both LABELLED as predicted, neither measured:

1. extrapolated measurements: every candidate's measured n = 2 and n = 4
   latency per size (tools/tune_b200.py --raw) is extended to n = 8 along its
   schedule's step count -- chain / pipelined chain / direct are linear in
   the n - 1 hops or receivers, the binomial tree in ceil(log2 n) rounds,
   scatter-ring-allgather in ceil(log2 n) + n - 1 steps -- and the library's
   tuner (bcl::tune with a cost function: argmin, geometric-mean bounds,
   merged ranges, the reference tie-breaks) picks the winners;
2. the paper's model: Eq. 5 + the per-call constant a0 fitted to the measured
   chain latencies at n = 2 and n = 4 (a0 linear in the hop count, bandwidth
   at the middle-rank ceiling measured at n = 4), then bcl::tune with the
   analytical oracle at n = 8 (NetworkParams.call_overhead_s = a0).

  python tools/predict_n8.py RAW2.csv RAW4.csv OUT_EXTRAP.csv OUT_EQ5.csv
"""
import csv
import math
import sys

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_1707_09414_b200 as B  # noqa: E402


def load(path):
    out = {}
    for r in csv.DictReader(open(path)):
        if r.get("protocol", "auto") != "auto":
            continue
        key = (r["algorithm"], int(r["radix"]), int(r["chunk_bytes"]), int(r["bytes"]))
        out.setdefault(key, float(r["seconds"]))  # first measurement = the default transport
    return out


def steps(algo, n):
    if algo in ("chain_pipelined", "chain", "direct"):
        return n - 1
    if algo in ("knomial", "knomial_staged"):
        return math.ceil(math.log2(n))
    if algo == "scatter_ring_allgather":
        return math.ceil(math.log2(n)) + n - 1
    raise ValueError(algo)


def extrapolate(t2, t4, algo):
    s2, s4, s8 = steps(algo, 2), steps(algo, 4), steps(algo, 8)
    slope = (t4 - t2) / (s4 - s2)
    return max(t4, t4 + slope * (s8 - s4))


def fit_eq5_a0(raw, n):
    rows, y = [], []
    for (algo, _, c, m), t in raw.items():
        if algo != "chain_pipelined" or m < (1 << 20):
            continue
        k = -(-m // c) + n - 2
        rows.append([1.0, k, k * c])
        y.append(t)
    A, y = np.array(rows), np.array(y)
    coef, *_ = np.linalg.lstsq(A / y[:, None], np.ones_like(y), rcond=None)
    a0, ts, inv_b = (max(float(v), 1e-15) for v in coef)
    rel = np.abs(A @ np.array([a0, ts, inv_b]) - y) / y
    return a0, ts, 1.0 / inv_b, float(np.median(rel)), len(y)


def main():
    raw2, raw4 = load(sys.argv[1]), load(sys.argv[2])
    sizes = [4 << i for i in range(29)]
    chunks = [65536 << i for i in range(7)]
    cands = [B.AlgorithmConfig.of("direct"), B.AlgorithmConfig.of("knomial", 2),
             B.AlgorithmConfig.of("scatter_ring_allgather"), B.AlgorithmConfig.of("chain_pipelined")]
    missing = []

    def at(raw, cfg, m):
        """Measured latency of cfg at m; between swept sizes (the tuner's
        merged-range midpoints) log-log interpolated between the neighbours."""
        key = (cfg.algorithm.name, cfg.radix_k, cfg.chunk_bytes)
        pts = sorted((mm, t) for (a, r, c, mm), t in raw.items() if (a, r, c) == key)
        if not pts:
            return None
        for (m0, t0), (m1, t1) in zip(pts, pts[1:]):
            if m0 <= m <= m1:
                if m == m0:
                    return t0
                f = math.log(m / m0) / math.log(m1 / m0)
                return math.exp(math.log(t0) + f * (math.log(t1) - math.log(t0)))
        if m > pts[-1][0]:  # above the sweep (the last range's midpoint): bandwidth-bound, linear in M
            return pts[-1][1] * m / pts[-1][0]
        return dict(pts).get(m)

    def cost(cfg, n, m):
        t2, t4 = at(raw2, cfg, m), at(raw4, cfg, m)
        if t2 is None or t4 is None:
            missing.append((cfg, m))
            return 1.0  # never measured at both n: never the winner
        return extrapolate(t2, t4, cfg.algorithm.name)

    t1 = B.tune_measured([8], sizes, cands, chunks, cost,
                         provenance="PREDICTED n=8, not measured: per-candidate B200 latencies measured at n=2 and "
                                    "n=4 (tools/tune_b200.py --raw) extrapolated along each schedule's step count "
                                    "(tools/predict_n8.py)")
    text = t1.text()
    lines = text.splitlines()
    lines.insert(1, "# bcl-predicted: n=8 (no 8-GPU box; gpurun grants at most 4 GPUs)")
    open(sys.argv[3], "w").write("\n".join(lines) + "\n")
    print(f"extrapolated table ({len(missing)} candidate points lacked a measurement at n=2 or n=4):")
    print("\n".join(lines))

    a2, ts2, b2, e2, k2 = fit_eq5_a0(raw2, 2)
    a4, ts4, b4, e4, k4 = fit_eq5_a0(raw4, 4)
    a8 = a4 + (a4 - a2) * (7 - 3) / (3 - 1)  # a0 linear in the hop count
    ts8, b8 = max(ts4, 1e-9), b4               # middle ranks set the bandwidth from n = 3 on
    print(f"\nEq. 5 + a0 fits (chain_pipelined, M >= 1 MiB): n=2 a0={a2*1e6:.2f} us t_s={ts2*1e6:.3f} us "
          f"B={b2/1e9:.0f} GB/s (median error {e2:.1%}, {k2} points); n=4 a0={a4*1e6:.2f} us "
          f"t_s={ts4*1e6:.3f} us B={b4/1e9:.0f} GB/s (median error {e4:.1%}, {k4} points)")
    print(f"n=8 parameters: a0={a8*1e6:.2f} us, t_s={ts8*1e6:.3f} us, B={b8/1e9:.0f} GB/s")
    t2 = B.tune([8], sizes, cands, chunks, startup_s=ts8, link_Bps=b8, call_overhead_s=a8)
    text = t2.text()
    lines = text.splitlines()
    lines.insert(1, f"# bcl-predicted: n=8 by the paper's Eq. 5 + a0 (a0 {a8*1e6:.2f} us, t_s {ts8*1e6:.3f} us, "
                    f"B {b8/1e9:.0f} GB/s) fitted to measured n=2/4 chain latencies; not measured")
    open(sys.argv[4], "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
