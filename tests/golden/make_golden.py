#!/usr/bin/env python3
"""Generate the golden fixtures from the REFERENCE itself.

Runs oracle/_ref/ref_harness (the unmodified bcastlab sources from
/root/reference/proj compiled by oracle/Makefile, plus our thin driver
oracle/ref_harness.cpp) and records its outputs as small JSON fixtures.
The fixtures pin both the C oracle (oracle/bcast_oracle.c) and the product
library; they are committed so the GPU box (no /root/reference) can use them.

Usage:  make -C oracle ref && python tests/golden/make_golden.py
"""
import json
import os
import random
import subprocess
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
HARNESS = os.path.join(ROOT, "oracle", "_ref", "ref_harness")

ALGOS = ["direct", "chain", "knomial", "scatter_ring_allgather",
         "chain_pipelined", "knomial_staged"]


def run(*args):
    out = subprocess.run([HARNESS, *map(str, args)], check=True,
                         capture_output=True, text=True).stdout
    return out


def schedule_cases():
    # Hand-picked goldens mirroring proj/tests/test_schedules.cpp, then a
    # seeded random sweep (rotation / validity property cases).
    cases = [
        ("direct", 3, 0, 100, 0, 0), ("direct", 3, 1, 100, 0, 0),
        ("chain", 3, 0, 100, 0, 0), ("chain", 4, 2, 100, 0, 0),
        ("knomial", 4, 0, 100, 0, 2), ("knomial", 2, 0, 100, 0, 2),
        ("knomial", 9, 0, 900, 0, 3), ("knomial", 8, 0, 64, 0, 2),
        ("knomial", 8, 5, 64, 0, 2),
        ("scatter_ring_allgather", 2, 0, 10, 0, 0),
        ("scatter_ring_allgather", 4, 0, 8, 0, 0),
        ("scatter_ring_allgather", 4, 0, 10, 0, 0),
        ("scatter_ring_allgather", 8, 0, 64, 0, 0),
        ("scatter_ring_allgather", 8, 3, 8192, 0, 0),
        ("scatter_ring_allgather", 5, 2, 3, 0, 0),
        ("chain_pipelined", 3, 0, 8, 4, 0), ("chain_pipelined", 5, 1, 100, 1000, 0),
        ("chain_pipelined", 4, 0, 64, 16, 0), ("chain_pipelined", 4, 0, 0, 16, 0),
        ("chain_pipelined", 8, 7, 1000, 999, 0), ("chain_pipelined", 2, 1, 10, 3, 0),
        ("knomial_staged", 8, 0, 4096, 0, 2),
    ]
    rng = random.Random(3)
    for _ in range(60):
        n = 1 + rng.randrange(16)
        root = rng.randrange(n)
        m = rng.randrange(10000)
        k = 2 + rng.randrange(4)
        chunk = 1 + rng.randrange(2048)
        algo = rng.choice(ALGOS)
        if algo == "chain_pipelined":
            if n < 2:
                n = 2
                root = rng.randrange(n)
            chunk = max(chunk, m // 40 + 1)  # keep fixtures small
        cases.append((algo, n, root, m, chunk, k))
    return cases


def parse_schedule(text):
    chunks, events, prologue = [], [], 0
    for line in text.splitlines():
        f = line.split()
        if f[0] == "prologue":
            prologue = int(f[1])
        elif f[0] == "chunk":
            chunks.append([int(f[1]), int(f[2]), int(f[3])])
        elif f[0] == "event":
            events.append([int(f[1]), 0 if f[2] == "send" else 1, int(f[3]),
                           int(f[4]), int(f[5])])
    return {"prologue": prologue, "chunks": chunks, "events": events}


def bcast_cases():
    cases = [
        # proj/tests/test_runtime.cpp:99-108 shape
        ("chain_pipelined", 4, 0, 64, 16, 0, 42),
        ("chain", 1, 0, 128, 0, 0, 1),
        ("knomial_staged", 8, 5, 4096, 0, 2, 3),
        ("scatter_ring_allgather", 8, 0, 8192, 0, 0, 7),
        ("knomial", 6, 0, 0, 0, 2, 0),
        ("chain_pipelined", 4, 0, 67108864 // 64, 524288 // 64, 0, 1),
    ]
    # acceptance.cpp:190-233 distribution (n in [2,16], M in [0, 1 MiB],
    # chunk in [1, M+1], radix in [2,4]); our own seeded draw.
    rng = random.Random(20260810)
    for trial in range(100):
        algo = ALGOS[trial % len(ALGOS)]
        n = 2 + rng.randrange(15)
        root = rng.randrange(n)
        m = rng.randrange(1048576 + 1) if trial % 5 else rng.randrange(64)
        radix = 2 + rng.randrange(3)
        chunk = 1 + rng.randrange(m + 1)
        if algo == "chain_pipelined" and (m + chunk - 1) // chunk > 4096:
            chunk = m // 4096 + 1
        cases.append((algo, n, root, m, chunk, radix, rng.randrange(1 << 30)))
    return cases


def tune_cases():
    return [
        # (n_list, lo, hi, candidates, chunk_lo, chunk_hi, oracle)
        ("4,8,16", 1024, 4194304, "knomial,chain_pipelined", 8192, 4194304, "analytical"),
        ("4", 1024, 4194304, "knomial,chain_pipelined", 8192, 4194304, "analytical"),
        ("2,4,8", 4, 1 << 30, "knomial,scatter_ring_allgather,chain_pipelined",
         65536, 4194304, "analytical"),
        ("4,8", 1024, 1048576, "chain", 8192, 8192, "analytical"),
        ("8,16", 1024, 1 << 26, "knomial,chain_pipelined", 8192, 4194304, "analytical"),
        ("4,8", 8192, 262144, "knomial,chain_pipelined", 8192, 4194304, "simulated"),
    ]


def main():
    out = {}
    sch = []
    for c in schedule_cases():
        algo, n, root, m, chunk, radix = c
        sch.append({"case": list(c), **parse_schedule(run("schedule", algo, n, root, m, chunk, radix))})
    out["schedules"] = sch

    bc = []
    for c in bcast_cases():
        algo, n, root, m, chunk, radix, seed = c
        text = run("bcast", algo, n, root, m, chunk, radix, seed, "inproc")
        lines = text.split("\n")
        payload = lines[0].split()[1]
        ranks = [l.split()[2] for l in lines[1:] if l.startswith("rank")]
        bc.append({"case": list(c), "payload_fnv": payload, "rank_fnv": ranks})
    out["bcasts"] = bc

    tables = []
    for c in tune_cases():
        text = run("tune", *c)
        tables.append({"case": list(c), "csv": text})
    out["tables"] = tables

    # select answers on the reference's own tables (tuner.cpp:178-197).
    sel = []
    rng = random.Random(99)
    for t in tables:
        with tempfile.NamedTemporaryFile("w", suffix=".csv", delete=False) as f:
            f.write(t["csv"])
            path = f.name
        probes = [0, 1, 3, 1023, 1024, 4096, 65536, 4194304, 8388607, 8388608,
                  1 << 30, (1 << 31) + 5] + [rng.randrange(1 << 32) for _ in range(40)]
        for n in (1, 2, 3, 4, 5, 8, 9, 16, 64, 128):
            res = run("select", path, n, *probes).splitlines()
            sel.append({"table": tables.index(t), "n": n, "probes": probes, "answers": res})
        os.unlink(path)
    out["selects"] = sel

    # Malformed tables (tuner.cpp:267-345 / test_tuner.cpp:230-265).
    hdr = "n,msg_min_bytes,msg_max_bytes,algorithm,radix,chunk_bytes,predicted_cost_s\n"
    bad = [hdr, hdr + "4,1024,2048,knomial,2,0\n", hdr + "4,1024,2048,ring,0,0,1e-5\n",
           hdr + "4,1024,4096,knomial,2,0,1e-5\n4,2048,8192,chain,0,0,2e-5\n",
           "garbage\n", "# oracle: magic\n" + hdr, "# oracle: simulated\n" + hdr + "4,1,2,chain,0,0,1\n",
           hdr + "0,1,2,chain,0,0,1\n", hdr + "4,5,5,chain,0,0,1\n",
           hdr + "4,1,2,chain,0,0,abc\n", hdr + "4,+1,2,chain,0,0,1\n",
           hdr + "4,1,2,chain,0,0,1,\n", "\n\n# comment\n" + hdr + "\r\n4,1,2,chain,0,0,1\r\n",
           hdr + "5,1,2,chain,0,0,1\n4,1,2,chain,0,0,1\n4,2,9,knomial,2,0,1e-3\n", ""]
    parsed = []
    for text in bad:
        with tempfile.NamedTemporaryFile("w", suffix=".csv", delete=False) as f:
            f.write(text)
            path = f.name
        res = run("select", path, 4, 1, 3).splitlines()
        parsed.append({"text": text, "result": res})
        os.unlink(path)
    out["parse"] = parsed

    models = []
    for n, m, c in [(4, 1000000, 125000), (16, 1024, 1024), (8, 67108864, 524288),
                    (2, 0, 1), (8, 1 << 30, 4194304)]:
        vals = dict(l.split() for l in run("models", n, m, c).splitlines())
        models.append({"n": n, "m": m, "c": c, "costs": {k: float(v) for k, v in vals.items()}})
    out["models"] = models

    path = os.path.join(HERE, "reference_golden.json")
    with open(path, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
