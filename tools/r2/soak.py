#!/usr/bin/env python3
"""Soak run (one process driving every visible GPU): random broadcasts across
every transport -- protocol auto/pull/push/ll/ll128/nvls, every schedule,
random roots, sizes from 1 B to 24 MiB, misaligned views, grouped runs of
2-8 calls, device barriers, and a captured CUDA graph replayed between them
-- every byte of every rank checked after each step.

  python tools/r2/soak.py [steps] [seed]
"""
import os
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402
import paper_1707_09414_b200 as B  # noqa: E402

ALGOS = ["chain_pipelined", "direct", "knomial", "scatter_ring_allgather", "chain"]


def cfg_of(algo, chunk):
    a = B.Algorithm[algo]
    return B.AlgorithmConfig(a, 2 if a == B.Algorithm.knomial else 0, chunk if a == B.Algorithm.chain_pipelined else 0)


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 500
    rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
    devices = list(range(torch.cuda.device_count()))
    n = len(devices)
    comms = B.Comm.local(devices, timeout_s=20)
    protos = ["auto", "pull", "push", "ll", "ll128"] + (["nvls"] if comms[0].nvls()[0] else [])
    cap = 24 << 20
    bufs = [torch.empty(cap + 64, dtype=torch.uint8, device=f"cuda:{d}") for d in devices]
    streams = [torch.cuda.Stream(device=f"cuda:{d}") for d in devices]
    # a captured graph: two broadcasts on fixed views, replayed between steps
    gviews = [[torch.zeros(m, dtype=torch.uint8, device=f"cuda:{d}") for d in devices] for m in (3000, (2 << 20) + 7, (1 << 20) + 5)]

    def graph_body():
        for k, v in enumerate(gviews):
            B.bcast_all(comms, v, v[0].numel(), "uint8", k % n, None, streams=streams)

    graph_body()
    for d in devices:
        torch.cuda.synchronize(d)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=streams[0]):
        start = torch.cuda.Event()
        start.record(streams[0])
        for st in streams[1:]:
            st.wait_event(start)
        graph_body()
        for st in streams[1:]:
            e = torch.cuda.Event()
            e.record(st)
            streams[0].wait_event(e)
    for d in devices:
        torch.cuda.synchronize(d)
    counts = {}
    for it in range(steps):
        proto = rng.choice(protos)
        for c in comms:
            c.set_protocol(proto)
        group = rng.random() < 0.3
        calls = rng.randint(2, 8) if group else 1
        plan = []
        at = 0
        for _ in range(calls):
            m = rng.choice([rng.randrange(1, 4097), rng.randrange(4097, 1 << 20), rng.randrange(1 << 20, 6 << 20)])
            if at + m + 16 > cap:
                break
            off = at + rng.randrange(0, 16)
            root = rng.randrange(n)
            algo = "chain_pipelined" if proto in ("ll", "ll128") else rng.choice(ALGOS)
            if proto == "ll" and m > (8 << 20):
                m = 8 << 20
            if algo in ("knomial", "scatter_ring_allgather", "chain") and proto == "nvls":
                pass
            plan.append((off, m, root, algo, rng.choice([4096, 65536, 262144, 1 << 20])))
            at = off + m
        srcs = []
        for off, m, root, algo, chunk in plan:
            src = torch.randint(0, 256, (m,), dtype=torch.uint8, device=f"cuda:{devices[root]}")
            for r in range(n):
                v = bufs[r][off:off + m]
                (v.copy_(src) if r == root else v.fill_(it & 0xFF))
            srcs.append(src)
        for d in devices:
            torch.cuda.synchronize(d)
        try:
            if group:
                with B.group():
                    for off, m, root, algo, chunk in plan:
                        B.bcast_all(comms, [b[off:off + m] for b in bufs], m, "uint8", root, cfg_of(algo, chunk),
                                    streams=streams)
            else:
                off, m, root, algo, chunk = plan[0]
                B.bcast_all(comms, [b[off:off + m] for b in bufs], m, "uint8", root, cfg_of(algo, chunk),
                            streams=streams)
        except ValueError as e:  # a protocol that cannot carry this call (e.g. LL above its cap): skip
            for c in comms:
                c.set_protocol("auto")
            counts["refused"] = counts.get("refused", 0) + 1
            continue
        if rng.random() < 0.2:
            B.barrier_all(comms, streams=streams)
        if rng.random() < 0.25:  # replay the captured graph (fresh payloads first)
            for k, v in enumerate(gviews):
                for r in range(n):
                    v[r].fill_((it + k) % 250 + 3 if r == k % n else 0)
            for d in devices:
                torch.cuda.synchronize(d)
            for c in comms:
                c.set_protocol("auto")  # the graph was captured under auto
            with torch.cuda.stream(streams[0]):
                g.replay()
            for d in devices:
                torch.cuda.synchronize(d)
            for k, v in enumerate(gviews):
                for r in range(n):
                    want = (it + k) % 250 + 3
                    assert int(v[r].min()) == want == int(v[r].max()), ("graph", it, k, r)
            counts["graph"] = counts.get("graph", 0) + 1
        for d in devices:
            torch.cuda.synchronize(d)
        for (off, m, root, algo, chunk), src in zip(plan, srcs):
            for r in range(n):
                if not torch.equal(bufs[r][off:off + m], src.to(f"cuda:{devices[r]}")):
                    raise SystemExit(f"MISMATCH step {it} proto {proto} algo {algo} m {m} root {root} rank {r}")
        key = f"{proto}{'/group' if group else ''}"
        counts[key] = counts.get(key, 0) + len(plan)
    for c in comms:
        c.check()
    print(f"soak ok: {steps} steps on {n} GPUs, every byte checked; messages per transport: {dict(sorted(counts.items()))}")


if __name__ == "__main__":
    main()
