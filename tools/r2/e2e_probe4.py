#!/usr/bin/env python3
"""Dev probe: where the N=1 host-buffer broadcast (64 MiB H2D + 3 x 64 MiB
D2H) loses against the PCIe floor -- raw copy shapes, then run_bcast_host
per host_piece."""
import os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1707_09414_b200 as B
m, n = 64 << 20, 4
dev = torch.device("cuda:0")
scr = [torch.empty(m, dtype=torch.uint8, device=dev) for _ in range(n)]
h = [torch.empty(m, dtype=torch.uint8, pin_memory=True) for _ in range(n)]
h[0].random_(0, 256)
st = [torch.cuda.Stream() for _ in range(4)]


def timed(fn, reps=6, zero=False):
    ts = []
    for _ in range(reps):
        if zero:
            for r in range(1, n):
                h[r].zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts[1:])


def d2h_one_stream():
    with torch.cuda.stream(st[0]):
        for r in range(1, n):
            h[r].copy_(scr[r], non_blocking=True)


def d2h_three_streams():
    for r in range(1, n):
        with torch.cuda.stream(st[r]):
            h[r].copy_(scr[r], non_blocking=True)


def h2d_and_d2h():
    with torch.cuda.stream(st[0]):
        scr[0].copy_(h[0], non_blocking=True)
    with torch.cuda.stream(st[1]):
        for r in range(1, n):
            h[r].copy_(scr[r], non_blocking=True)


def d2h_pieces(piece):
    def f():
        with torch.cuda.stream(st[0]):
            for off in range(0, m, piece):
                for r in range(1, n):
                    h[r][off:off + piece].copy_(scr[r][off:off + piece], non_blocking=True)
    return f


for name, fn in [("D2H 3x64 MiB one stream", d2h_one_stream), ("D2H 3x64 MiB three streams", d2h_three_streams),
                 ("H2D 64 MiB || D2H 3x64 MiB", h2d_and_d2h)] + \
        [(f"D2H in {p >> 20} MiB pieces", d2h_pieces(p)) for p in (1 << 20, 4 << 20, 16 << 20)]:
    t = timed(fn)
    print(f"{name}: {t * 1e3:.3f} ms", flush=True)

cfg = B.AlgorithmConfig(B.Algorithm.chain_pipelined, 0, 512 << 10)
comms = B.Comm.local([0] * n, timeout_s=30)


def pipeline(piece, use_bcast):
    def f():
        for off in range(0, m, piece):
            ln = min(piece, m - off)
            with torch.cuda.stream(st[0]):
                scr[0][off:off + ln].copy_(h[0][off:off + ln], non_blocking=True)
            st[1].wait_stream(st[0])
            if use_bcast:
                B.bcast_all(comms, [x[off:off + ln] for x in scr], ln, "uint8", 0, cfg, streams=[st[1]] * n)
            else:
                with torch.cuda.stream(st[1]):
                    for r in range(1, n):
                        scr[r][off:off + ln].copy_(scr[0][off:off + ln], non_blocking=True)
            st[2].wait_stream(st[1])
            with torch.cuda.stream(st[2]):
                for r in range(1, n):
                    h[r][off:off + ln].copy_(scr[r][off:off + ln], non_blocking=True)
    return f


for piece in (4 << 20, 8 << 20):
    for use in (False, True):
        for zero in (False, True):
            t = timed(pipeline(piece, use), zero=zero)
            print(f"python pipeline piece {piece >> 20} MiB {'bcast_all' if use else 'd2d copies'}"
                  f"{' (host buffers zeroed by the CPU first)' if zero else ''}: {t * 1e3:.3f} ms", flush=True)
t = timed(d2h_one_stream, zero=True)
print(f"D2H 3x64 MiB one stream, host buffers zeroed first: {t * 1e3:.3f} ms", flush=True)
for piece in (2 << 20, 4 << 20, 8 << 20, 16 << 20):
    for extra in ("", "split"):
        opts = {"host_piece": piece}
        if extra:
            os.environ["BCL_HOST_SPLIT_D2H"] = "1"
        cs = B.Comm.local([0] * n, timeout_s=30, **opts)
        ws, wz = [], []
        for it in range(7):
            ws.append(B.run_bcast_host(cs, 0, h, m, cfg))
        for it in range(7):
            for r in range(1, n):
                h[r].zero_()
            wz.append(B.run_bcast_host(cs, 0, h, m, cfg))
        print(f"  (zeroed first: {statistics.median(wz[1:]) * 1e3:.3f} ms)", flush=True)
        ok = all(torch.equal(h[r], h[0]) for r in range(1, n))
        print(f"run_bcast_host piece {piece >> 20} MiB {extra or 'one D2H stream'}: "
              f"{statistics.median(ws[1:]) * 1e3:.3f} ms ({m / statistics.median(ws[1:]) / 1e9:.1f} GB/s) ok={ok}",
              flush=True)
        os.environ.pop("BCL_HOST_SPLIT_D2H", None)
        for c in cs:
            c.close()
