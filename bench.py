#!/usr/bin/env python3
"""Benchmark of the B200 pipelined-chain broadcast (BASELINE.json metric:
bcast latency & bus GB/s vs message size, vs ncclBroadcast).

  python bench.py [--steps K] [--warmup W]                      N=1
  torchrun --nproc-per-node N bench.py --gpus N [...]           N>1, one rank per GPU
  python bench.py --impl reference [...]                        the reference CPU path

Workloads
  N=1  BASELINE config 1 (the reference's CPU case): 4 ranks, 64 MiB float32,
       root 0, 512 KiB chunks, pipelined chain — the 4 ranks share cuda:0 and
       run in one cooperative launch, so every hop is an HBM read+write.
  N>1  the same 64 MiB / 512 KiB pipelined chain over N GPUs (one process
       each, buffers in the CUDA-IPC symmetric heap, pulls over NVLink), plus
       the 4 B - 1 GiB sweep with the tuned algorithm per size next to
       ncclBroadcast (called directly on the same stream and buffers).

Method (osu_bcast as bcastlab bench, proj/tools/bcastlab.cpp:147-206): per
step non-root buffers are zeroed, L2 is flushed (256 MiB read), ranks meet
at a device barrier, the broadcast is timed with CUDA events on its stream,
every buffer is verified before the time is kept; per-step latency is the
max over ranks. One JSON line on rank 0.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS = {}
try:
    PEAKS = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
except OSError:
    pass
HBM_PEAK = float(PEAKS.get("hbm_gbs", 6650.0))
try:  # DRAM bytes per launch of the N=1 kernel from the committed ncu --set full capture
    TRAFFIC_N1 = json.load(open(os.path.join(ROOT, "profiles", "round2", "n1", "ncu_traffic.json")))[
        "n1_config1_local_chain_kernel"]["dram_bytes_per_launch"]
except (OSError, KeyError, ValueError):
    TRAFFIC_N1 = None
HBM_PEAK_SRC = "measured" if "hbm_gbs" in PEAKS else "fallback"
LINK_BW = 900e9  # north_star chain roofline: NVLink-5 per direction per GPU
NVLINK_MEASURED = 770.0  # GB/s per direction, peer copy measured on this pool (B200_PROFILING.md)
try:  # NVLink bytes per launch of the cross-GPU kernels, ncu (profiles/round2/xgpu/, tools/r2/ncu_xgpu.py)
    XGPU = json.load(open(os.path.join(ROOT, "profiles", "round2", "xgpu", "ncu_xgpu_traffic.json")))
except (OSError, ValueError):
    XGPU = None


def nvlink_traffic(path, m, world):
    """NVLink bytes one receiving GPU takes in per call of the dominant kernel,
    from the committed ncu capture of that kernel (nvlrx/nvltx__bytes; NVML
    exposes no NVLink counters on this pool: NOT_SUPPORTED). Exact for the
    captured shape, scaled by the measured bytes-per-payload-byte otherwise."""
    if XGPU is None:
        return None, "no ncu capture committed"
    if path.startswith("bcast_kernel/pull"):
        k = XGPU["pull_receiver_n2_64MiB"]
        exact = m == 64 << 20 and world == 2
        t = k["nvlink_rx_bytes"] if exact else k["nvlink_rx_bytes"] / k["nvlink_rx_user_bytes"] * m
        return round(t), ("ncu nvlrx__bytes.sum of the receiver's bcast_kernel, N=2 64 MiB (%s); user data "
                          "%d B = M, the rest request/response protocol" % ("this shape" if exact else "scaled to M",
                                                                            k["nvlink_rx_user_bytes"]))
    if path == "ll128_kernel":
        k = XGPU["ll128_n2_32MiB"][0]
        t = k["nvlink_tx_bytes"] / 33554432 * m
        return round(t), ("ncu nvltx__bytes.sum of the LL128 writer per payload byte (N=2, 32 MiB capture) x M: "
                          "128-byte lines carry 120 payload bytes, plus protocol")
    return None, "no ncu capture of %s" % path
METRIC = "bcast latency (us) & bus GB/s vs msg size 4B–1GB at 2/4/8 B200 vs ncclBroadcast"


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: NVML polled
    every 2 ms from a thread (nvidia-smi's first sample arrives only after the
    short timed regions here have ended); nvidia-smi -lms as the fallback."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, gpu):
        self.gpu, self.sm, self.mx, self.reasons, self.stop = gpu, [], [], set(), threading.Event()
        self.t = None

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.gpu]) if vis and vis.split(",")[self.gpu].isdigit() else self.gpu
            h = nv.nvmlDeviceGetHandleByIndex(idx)
            self.mx.append(float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)))

            def poll():
                while not self.stop.is_set():
                    self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                    bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    for name, const in self.REASONS:
                        if bits & getattr(nv, const):
                            self.reasons.add(name)
                    time.sleep(0.002)
            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            while not self.sm and self.t.is_alive():  # first sample before the region starts
                time.sleep(0.0005)
        except Exception:  # noqa: BLE001 - no NVML: report unsampled
            self.t = None
        return self

    def __exit__(self, *exc):
        self.stop.set()
        if self.t:
            self.t.join(timeout=2)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": max(self.mx) if self.mx else None,
                "reasons": sorted(self.reasons), "samples": len(self.sm)}


class NcclDirect:
    """ncclBroadcast called directly (nccl-tests style) on our stream and our
    buffers: the NCCL torch bundles (libnccl.so.2), its own communicator
    (unique id shared over torch.distributed), no ProcessGroup stream hop."""

    def __init__(self, torch, rank, world):
        import ctypes as C
        import torch.distributed as dist
        path = None
        try:
            import nvidia.nccl
            path = os.path.join(list(nvidia.nccl.__path__)[0], "lib", "libnccl.so.2")
        except ImportError:
            pass
        self.C = C
        self.lib = C.CDLL(path if path and os.path.exists(path) else "libnccl.so.2")

        class UniqueId(C.Structure):
            _fields_ = [("internal", C.c_ubyte * 128)]
        uid = UniqueId()
        if rank == 0:
            self._ok(self.lib.ncclGetUniqueId(C.byref(uid)))
        blob = [C.string_at(C.addressof(uid), 128) if rank == 0 else None]  # all 128 bytes (NULs included)
        dist.broadcast_object_list(blob, src=0)
        C.memmove(C.addressof(uid), blob[0], 128)
        self.comm = C.c_void_p()
        self._ok(self.lib.ncclCommInitRank(C.byref(self.comm), world, uid, rank))
        v = C.c_int()
        self.lib.ncclGetVersion(C.byref(v))
        self.version = v.value
        self.lib.ncclBroadcast.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_void_p,
                                           C.c_void_p]

    def _ok(self, r):
        if r != 0:
            raise RuntimeError(f"NCCL error {r}")

    def bcast(self, buf, nbytes, root, stream):
        p = buf.data_ptr()
        self._ok(self.lib.ncclBroadcast(p, p, nbytes, 1, root, self.comm, stream.cuda_stream))  # ncclUint8

    def close(self):
        if self.comm:
            self.lib.ncclCommDestroy(self.comm)
            self.comm = None


def host_cpu():
    """Host core count and CPU model of this box (for the CPU baseline)."""
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "model": model}


def verdict(ours, theirs, tie=0.03):
    """win / tie / loss on medians; within 3% is a tie."""
    if ours <= theirs * (1 - tie):
        return "win"
    if ours >= theirs * (1 + tie):
        return "loss"
    return "tie"


# ----------------------------------------------------------------- CPU legs

def reference_cpu(n, m, chunk, iters, warmup=1, seed=1):  # noqa: C901
    """The reference's own CPU broadcast (oracle/_ref, unmodified bcastlab
    sources) timed with the osu method on this host: n rank threads."""
    harness = os.path.join(ROOT, "oracle", "_ref", "ref_harness")
    if os.path.exists(harness):
        out = subprocess.run([harness, "bench", "chain_pipelined", str(n), "0", str(m), str(chunk), "0",
                              str(warmup), str(iters), "inproc", str(seed)],
                             capture_output=True, text=True, check=True).stdout
        r = json.loads(out)
        return {"median_s": r["median_us"] * 1e-6, "min_s": r["min_us"] * 1e-6, "cores": n, "kind": "reference",
                "ok": r["ok"], "iters": iters,
                "sample": f"{iters} timed iterations (+{warmup} warm-up) of the full workload, inproc transport"}
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import _oracle as O  # the plain-C restatement (single thread)
    payload = O.payload(seed, m)
    times = []
    for _ in range(iters):
        bufs = [bytearray(m) for _ in range(n)]
        bufs[0][:] = payload
        t0 = time.perf_counter()
        O.bcast("chain_pipelined", n, 0, bufs, chunk=chunk)
        times.append(time.perf_counter() - t0)
    return {"median_s": statistics.median(times), "min_s": min(times), "cores": 1, "kind": "port", "ok": True,
            "iters": iters, "sample": f"{iters} iterations of the full workload through the C oracle port"}


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    n = 4 if world == 1 else world
    m, chunk = args.bytes, args.chunk
    iters = max(1, args.steps)
    r = reference_cpu(n, m, chunk, iters, warmup=max(1, min(args.warmup, 2)))
    v = m / r["median_s"] / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": "GB/s", "n_gpus": world,
            "steps": iters, "warmup": args.warmup, "ms_per_step": round(r["median_s"] * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": workload_config(n, m, chunk, world),
            "cpu_baseline": {"value": round(v, 4), "unit": "GB/s", "cores": r["cores"], "kind": r["kind"],
                             "sample": r["sample"]},
            "e2e": {"value": round(v, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "correct": r["ok"]}
    print(json.dumps(line), flush=True)


def workload_config(n, m, chunk, world):
    if world == 1:
        wl = (f"BASELINE config 1: pipelined-chain bcast, {n} ranks sharing one B200 (one launch; every hop "
              f"copies each chunk from the previous rank's buffer, hops fused per item), "
              f"{m >> 20} MiB float32 payload, root 0, {chunk >> 10} KiB chunks")
    else:
        wl = (f"bcast over {world} B200 (one process per GPU, NVLink P2P), {m >> 20} MiB float32, root 0, "
              f"tuner-selected algorithm/chunk; sweep 4 B-1 GiB vs NCCL")
    return {"workload": wl, "ranks": n, "bytes": m, "chunk_bytes": chunk, "root": 0,
            "algorithm": "chain_pipelined", "l2": "flushed between steps (256 MiB read sweep)"}


# ----------------------------------------------------------------- GPU legs

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--bytes", type=int, default=64 << 20)
    ap.add_argument("--chunk", type=int, default=512 << 10)
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--b2b-max", type=int, default=1 << 20,
                    help="N>1 sweep: also time 50 back-to-back calls up to this size")
    ap.add_argument("--sweep-max", type=int, default=1 << 30)
    ap.add_argument("--cpu-iters", type=int, default=12)
    ap.add_argument("--workload", default="config1", choices=["config1", "vgg16", "alexnet", "resnet50", "lenet"],
                    help="config1 (default) or a layer-wise parameter broadcast (BASELINE configs 4/5)")
    ap.add_argument("--bucket", type=int, default=0, help="parameter workloads: coalesce tensors into >= this")
    ap.add_argument("--fused", action="store_true",
                    help="parameter workloads: issue the per-tensor broadcasts inside one bcl_group_start/end")
    ap.add_argument("--graph", action="store_true",
                    help="parameter workloads: capture one iteration's broadcasts (ours and NCCL's) in a CUDA graph "
                         "and replay it per step")
    ap.add_argument("--csv", default=None, help="N>1: write the sweep as the reference bench CSV here")
    ap.add_argument("--fixed-chunk", dest="tuned", action="store_false",
                    help="N>1: pipelined chain with --chunk instead of the tuned selection")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    import torch
    if args.workload != "config1":
        if world == 1:
            raise SystemExit("parameter workloads need >= 2 GPUs (torchrun)")
        bench_params(args, torch, rank, world)
    elif world == 1:
        bench_single(args, torch)
    else:
        bench_multi(args, torch, rank, world)


GATE_CYCLES = 1_000_000  # ~0.5 ms spin: the host enqueues the timed ops behind it


HOST_RESET_NOTE = ("receivers' host buffers zeroed before every step by a D2H copy of zeros (outside the timed "
                   "region); a CPU memset would leave them dirty in the CPU caches, which the broadcast's D2H "
                   "DMA then pays for (raw 192 MiB D2H 4.75 vs 3.55 ms, profiles/round2/n1/e2e_probe4.log)")


CPU_READ_NOTE = ("value: receivers' host bytes verified every step by DMA-ing them back and comparing on the "
                 "GPU; cpu_read_between_calls_ms: the same calls when the CPU reads the receivers' pages "
                 "between calls (verification on the CPU), which leaves them in the CPU caches and slows "
                 "the next D2H into them by ~2 ms (profiles/round2/n1/e2e_probe6.log)")


def host_reset(host, zeros):
    """Zero a pinned host buffer by DMA (see HOST_RESET_NOTE)."""
    host.copy_(zeros[:host.numel()])


def flush_l2(torch, flush):
    """Evict L2 with a READ sweep of 256 MiB: it writes back the previous
    step's dirty lines before the timed region and leaves only clean lines
    (a write sweep left ~126 MB of dirty lines to be written back inside it)."""
    torch.sum(flush)


def time_steps(torch, steps, warmup, prepare, body, verify, stream, align=None, gate=None):
    """Runs warmup+steps iterations; returns the per-step body times (s).

    Per step: prepare (buffer reset, L2 flush) -> a GPU-side gate
    (torch.cuda._sleep) so that everything after it is already enqueued when
    the GPU reaches it -> align (device barrier across ranks) -> ev0 -> body
    -> ev1. Host launch overhead therefore never lands inside [ev0, ev1]."""
    times = []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for it in range(warmup + steps):
        prepare(it)
        with torch.cuda.stream(stream):
            torch.cuda._sleep(gate or GATE_CYCLES)
        if align is not None:
            align()
        ev0.record(stream)
        body(it)
        ev1.record(stream)
        ev1.synchronize()
        if not verify(it):
            raise RuntimeError(f"verification failed at iteration {it}")
        if it >= warmup:
            times.append(ev0.elapsed_time(ev1) * 1e-3)
    return times


def bench_single(args, torch):
    import paper_1707_09414_b200 as B
    n, m, chunk = 4, args.bytes, args.chunk
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    comms = B.Comm.local([0] * n, timeout_s=30)
    cfg = B.AlgorithmConfig(B.Algorithm.chain_pipelined, 0, chunk)
    stream = torch.cuda.Stream()
    g = torch.Generator(device=dev).manual_seed(1)
    bufs = [torch.zeros(m, dtype=torch.uint8, device=dev) for _ in range(n)]
    bufs[0].copy_(torch.randint(0, 256, (m,), dtype=torch.uint8, device=dev, generator=g))
    flush = torch.ones(256 << 18, dtype=torch.int32, device=dev)  # 256 MiB > 126 MB L2
    torch.cuda.synchronize()  # setup ran on the default stream; the timed loop uses `stream`

    def prepare(it):
        with torch.cuda.stream(stream):
            for r in range(1, n):
                bufs[r].zero_()
            flush_l2(torch, flush)

    def body(it):
        B.bcast_all(comms, bufs, m, "uint8", 0, cfg, streams=[stream] * n)

    def verify(it):
        return all(torch.equal(bufs[r], bufs[0]) for r in range(1, n))

    launches0 = comms[0].launches
    torch.cuda.synchronize()
    with ClockSampler(0) as clk:
        times = time_steps(torch, args.steps, args.warmup, prepare, body, verify, stream)
    torch.cuda.synchronize()
    launches = comms[0].launches - launches0 - args.warmup

    t = statistics.mean(times)
    busbw = m / t / 1e9
    # Roofline of the dominant (only) kernel, local_chain_kernel: every hop
    # reads M and writes M, but hop h+1 re-reads what hop h just wrote (an L2
    # hit by construction), so the DRAM bytes the algorithm needs per launch
    # are P*M: the root's M read once plus (P-1) M written. 2(P-1)M bytes move
    # through L2 and are reported beside it.
    alg_bytes = n * m
    achieved = alg_bytes / t / 1e9

    # e2e through the C-ABI with pinned host buffers (run_bcast_host).
    hosts = [torch.empty(m, dtype=torch.uint8, pin_memory=True) for _ in range(n)]
    hosts[0].copy_(bufs[0])  # by DMA: no CPU-cached lines for the H2D to snoop (HOST_RESET_NOTE)
    zeros = torch.zeros(m, dtype=torch.uint8, device=dev)
    check = torch.empty(m, dtype=torch.uint8, device=dev)

    def e2e_loop(iters, cpu_verify):
        ts = []
        for it in range(iters):
            for r in range(1, n):
                host_reset(hosts[r], zeros)
            w = B.run_bcast_host(comms, 0, hosts, m, cfg)
            for r in range(1, n):  # verify before recording
                if cpu_verify:
                    ok = torch.equal(hosts[r], hosts[0])
                else:
                    check.copy_(hosts[r])  # the host bytes, DMA'd back and compared on the GPU
                    ok = torch.equal(check, bufs[0])
                if not ok:
                    raise RuntimeError("e2e verification failed")
            ts.append(w)
        return ts

    e2e = e2e_loop(args.warmup + max(3, args.steps // 2), False)[args.warmup:]
    e2e_t = statistics.mean(e2e)
    warm = e2e_loop(2 + max(3, args.steps // 4), True)[2:]  # receivers' pages read by the CPU between calls

    cpu = reference_cpu(n, m, chunk, args.cpu_iters)
    line = {
        "metric": METRIC, "value": round(busbw, 2), "unit": "GB/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(t * 1e3, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic (torch.randint bytes, float32-sized payload)",
        "config": workload_config(n, m, chunk, 1),
        "latency_us": {"mean": round(t * 1e6, 2), "min": round(min(times) * 1e6, 2),
                       "median": round(statistics.median(times) * 1e6, 2), "max": round(max(times) * 1e6, 2)},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": HBM_PEAK, "unit": "GB/s",
                     "frac": round(achieved / HBM_PEAK, 4), "traffic": TRAFFIC_N1 if m == 64 << 20 else None,
                     "algorithmic_bytes": alg_bytes, "l2_bytes": 2 * (n - 1) * m,
                     "l2_gbs": round(2 * (n - 1) * m / t / 1e9, 1),
                     "note": f"kernel local_chain_kernel; DRAM-algorithmic bytes P*M per launch (root read once, "
                             f"P-1 copies written; hop re-reads of the previous hop's output are L2 hits), "
                             f"2(P-1)M through L2; traffic = ncu DRAM bytes per launch, below P*M because the "
                             f"last writes are still in L2 when the kernel ends; peak {HBM_PEAK_SRC}"},
        "cpu_baseline": {"value": round(m / cpu["median_s"] / 1e9, 4), "unit": "GB/s", "cores": cpu["cores"],
                         "kind": cpu["kind"], "sample": cpu["sample"]},
        "e2e": {"value": round(m / e2e_t / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": m,
                "d2h_bytes_per_step": (n - 1) * m, "latency_ms": round(e2e_t * 1e3, 3),
                "path": "bcl_run_bcast_host (C-ABI), pinned host buffers", "reset": HOST_RESET_NOTE,
                "cpu_read_between_calls_ms": round(statistics.mean(warm) * 1e3, 3),
                "cpu_read_note": CPU_READ_NOTE},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def bench_multi(args, torch, rank, world):
    import torch.distributed as dist
    import paper_1707_09414_b200 as B
    from paper_1707_09414_b200.comm import DevicePtr
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    m, chunk = args.bytes, args.chunk
    sweep_max = args.sweep_max if not args.no_sweep else 0
    heap = max(m, sweep_max) + m + (16 << 20)
    comm = B.Comm.connect_torch(world, rank, local, heap_bytes=heap, timeout_s=30)
    stream = torch.cuda.Stream(device=dev)
    cap = max(m, sweep_max)
    raw = comm.alloc(cap)
    buf_all = torch.as_tensor(DevicePtr(raw, cap), device=dev)
    ref_all = torch.empty(cap, dtype=torch.uint8, device=dev)
    g = torch.Generator(device=dev).manual_seed(1)
    ref_all.copy_(torch.randint(0, 256, (cap,), dtype=torch.uint8, device=dev, generator=g))
    flush_buf = torch.ones(256 << 18, dtype=torch.int32, device=dev)
    nccl_direct = NcclDirect(torch, rank, world)
    torch.cuda.synchronize()  # setup ran on the default stream; the timed loop uses `stream`

    def run(size, steps, warmup, ours, cfg=None, flush=True):
        buf = buf_all[:size]
        ref = ref_all[:size]

        def prepare(it):
            with torch.cuda.stream(stream):
                if rank == 0:
                    buf.copy_(ref)
                else:
                    buf.zero_()
                if flush:
                    flush_l2(torch, flush_buf)
            if it == 0:
                stream.synchronize()
                dist.barrier(device_ids=[local])

        def body(it):
            if ours:
                comm.bcast(buf, size, "uint8", 0, cfg, stream=stream)
            else:
                nccl_direct.bcast(buf, size, 0, stream)

        def verify(it):
            return torch.equal(buf, ref)

        times = time_steps(torch, steps, warmup, prepare, body, verify, stream,
                           align=lambda: comm.barrier(stream))
        t = torch.tensor(times, dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ok = torch.tensor([1.0], device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        return t.cpu().tolist()

    def back_to_back(size, ours, calls=50):
        """Mean device time per call over `calls` back-to-back broadcasts
        between one pair of events (max over ranks); resolves what a single
        event pair cannot (~2 us ticks)."""
        buf = buf_all[:size]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for rep in range(2):  # warm, then timed
            stream.synchronize()
            dist.barrier(device_ids=[local])
            with torch.cuda.stream(stream):
                torch.cuda._sleep(GATE_CYCLES)
            comm.barrier(stream)
            e0.record(stream)
            for _ in range(calls):
                if ours:
                    comm.bcast(buf, size, "uint8", 0, None, stream=stream)
                else:
                    nccl_direct.bcast(buf, size, 0, stream)
            e1.record(stream)
            e1.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) * 1e-3 / calls], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        with torch.cuda.stream(stream):
            ok = torch.equal(buf, ref_all[:size])
        if not ok:
            raise RuntimeError("back-to-back verification failed")
        return float(t.item())

    # Headline: the configuration the tuner selects for this size (the
    # paper's framework picks algorithm and chunk); --chunk pins a chunk.
    cfg = comm.choose(m) if args.tuned else B.AlgorithmConfig(B.Algorithm.chain_pipelined, 0, chunk)
    dist.barrier(device_ids=[local])
    launches0 = comm.launches
    with ClockSampler(local) as clk:
        times = run(m, args.steps, args.warmup, True, cfg)
    launches = comm.launches - launches0 - args.warmup
    nccl = run(m, args.steps, args.warmup, False)

    # e2e through the C-ABI with pinned host buffers (bcl_bcast_host)
    host = torch.empty(m, dtype=torch.uint8, pin_memory=True)
    e2e = []
    zeros = torch.zeros(m, dtype=torch.uint8, device=dev)
    chk = torch.empty(m, dtype=torch.uint8, device=dev)
    for it in range(args.warmup + max(3, args.steps // 2)):
        if rank == 0:  # the root's payload lands in its host buffer by DMA too (HOST_RESET_NOTE)
            host.copy_(ref_all[:m])
        else:
            host_reset(host, zeros)
        dist.barrier(device_ids=[local])
        t0 = time.perf_counter()
        comm.bcast_host(host, m, "uint8", 0, cfg, stream=stream)
        stream.synchronize()
        w = time.perf_counter() - t0
        chk.copy_(host)  # the host bytes, DMA'd back and compared on the GPU (CPU_READ_NOTE)
        if not torch.equal(chk, ref_all[:m]):
            raise RuntimeError("e2e verification failed")
        wt = torch.tensor([w], dtype=torch.float64, device=dev)
        dist.all_reduce(wt, op=dist.ReduceOp.MAX)
        if it >= args.warmup:
            e2e.append(float(wt.item()))
    comm.reset_heap()
    raw = comm.alloc(cap)  # same region; the e2e scratch lived above it

    sweep = []
    nvls_ok, nvls_why = comm.nvls()
    if sweep_max:
        size = 4
        while size <= sweep_max:
            steps = 20 if size <= (16 << 20) else 8
            c = comm.choose(size)
            ours = run(size, steps, 3, True, None, flush=False)
            theirs = run(size, steps, 3, False, None, flush=False)
            to, tn = statistics.median(ours), statistics.median(theirs)
            b2b = None
            if size <= args.b2b_max:  # CUDA events tick every ~2 us here: average 50 back-to-back calls too
                bo, bn = back_to_back(size, True), back_to_back(size, False)
                b2b = {"ours_us": round(bo * 1e6, 3), "nccl_us": round(bn * 1e6, 3), "vs_nccl": verdict(bo, bn)}
            nv = None
            if nvls_ok and size >= 1024:  # NVLS multicast comparison point (north_star), protocol forced
                comm.set_protocol("nvls")
                tv = run(size, steps, 3, True, B.AlgorithmConfig(B.Algorithm.direct, 0, 0), flush=False)
                comm.set_protocol("auto")
                nv = {"min": round(min(tv) * 1e6, 2), "median": round(statistics.median(tv) * 1e6, 2),
                      "max": round(max(tv) * 1e6, 2), "busbw": round(size / statistics.median(tv) / 1e9, 2)}
            ch = c.chunk_bytes if c.algorithm == B.Algorithm.chain_pipelined else size
            t_roof = size / LINK_BW + (world - 1) * min(max(ch, 1), size) / LINK_BW
            sweep.append({"bytes": size, "algorithm": c.algorithm.name, "chunk": c.chunk_bytes,
                          "ours_us": {"min": round(min(ours) * 1e6, 2), "median": round(to * 1e6, 2),
                                      "max": round(max(ours) * 1e6, 2)},
                          "nccl_us": {"min": round(min(theirs) * 1e6, 2), "median": round(tn * 1e6, 2),
                                      "max": round(max(theirs) * 1e6, 2)},
                          "ours_busbw": round(size / to / 1e9, 2), "nccl_busbw": round(size / tn / 1e9, 2),
                          "frac_of_chain_roofline": round(t_roof / to, 4) if size >= (1 << 20) else None,
                          "vs_nccl": verdict(to, tn), "iterations": steps, "back_to_back": b2b,
                          "ours_mean_us": round(statistics.mean(ours) * 1e6, 2), "nvls_us": nv,
                          "path": comm.path(size, None)})
            size *= 2

    cpu = None
    if rank == 0:
        cpu = reference_cpu(world, m, cfg.chunk_bytes if cfg.algorithm == B.Algorithm.chain_pipelined else chunk,
                            max(3, args.cpu_iters // 2))
    dist.barrier(device_ids=[local])

    if rank == 0:
        t = statistics.mean(times)
        t_nccl = statistics.mean(nccl)
        busbw = m / t / 1e9
        t_roof = m / LINK_BW + (world - 1) * max(cfg.chunk_bytes, 1) / LINK_BW
        path = comm.path(m, cfg)
        traffic, traffic_note = nvlink_traffic(path, m, world)
        line = {
            "metric": METRIC, "value": round(busbw, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(t * 1e3, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic (torch.randint bytes)",
            "config": dict(workload_config(world, m, cfg.chunk_bytes, world), algorithm=cfg.algorithm.name,
                           selection="tuned (builtin measured table)" if args.tuned else "fixed"),
            "latency_us": {"mean": round(t * 1e6, 2), "min": round(min(times) * 1e6, 2),
                           "median": round(statistics.median(times) * 1e6, 2), "max": round(max(times) * 1e6, 2)},
            "nccl": {"busbw": round(m / t_nccl / 1e9, 2), "latency_us": round(t_nccl * 1e6, 2),
                     "median_us": round(statistics.median(nccl) * 1e6, 2), "vs_ours": verdict(t, t_nccl),
                     "impl": "ncclBroadcast called directly on the same stream and buffers (NCCL %d)"
                             % nccl_direct.version},
            "roofline": {"bound": "nvlink", "achieved": round(busbw, 1), "peak": LINK_BW / 1e9, "unit": "GB/s",
                         "frac": round(busbw / (LINK_BW / 1e9), 4),
                         "traffic": traffic, "traffic_note": traffic_note,
                         "kernel": path, "measured_peak_gbs": NVLINK_MEASURED,
                         "frac_of_measured_peak": round(busbw / NVLINK_MEASURED, 4),
                         "chain_roofline_us": round(t_roof * 1e6, 2), "frac_of_chain_roofline": round(t_roof / t, 4),
                         "note": "per-GPU ingress M/t vs NVLink-5 900 GB/s per direction (north_star)"},
            "cpu_baseline": {"value": round(m / cpu["median_s"] / 1e9, 4), "unit": "GB/s", "cores": cpu["cores"],
                             "kind": cpu["kind"], "sample": cpu["sample"], "host": host_cpu()},
            "e2e": {"value": round(m / statistics.mean(e2e) / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": m,
                    "d2h_bytes_per_step": (world - 1) * m, "latency_ms": round(statistics.mean(e2e) * 1e3, 3),
                    "path": "bcl_bcast_host (C-ABI) per rank, pinned host buffers", "reset": HOST_RESET_NOTE},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "sweep": sweep,
        }
        if sweep:
            line["sweep_vs_nccl"] = {k: sum(1 for e in sweep if e["vs_nccl"] == k) for k in ("win", "tie", "loss")}
            line["sweep_vs_nccl_back_to_back"] = {k: sum(1 for e in sweep if e["back_to_back"] and
                                                         e["back_to_back"]["vs_nccl"] == k)
                                                  for k in ("win", "tie", "loss")}
            line["nvls"] = {"available": nvls_ok, "reason": nvls_why or None,
                            "note": "nvls_us: the same broadcast forced onto the NVLS multicast path (protocol 5, "
                                    "direct schedule), single-call medians like ours_us"}
            line["sweep_note"] = ("single-call medians (osu method; CUDA events tick every ~2 us on this box, so "
                                  "differences under one tick are noise) and, up to 1 MiB, the mean of 50 "
                                  "back-to-back calls; within 3% = tie")
            csv_path = args.csv or (os.path.join("gpurun_out", f"bench_sweep_n{world}.csv")
                                    if os.path.isdir("gpurun_out") else None)
            if csv_path:
                write_bench_csv(csv_path, sweep)
        print(json.dumps(line), flush=True)
    dist.barrier(device_ids=[local])
    nccl_direct.close()
    comm.close()
    dist.destroy_process_group()


def write_bench_csv(path, sweep):
    """The reference bench's CSV (proj/tools/bcastlab.cpp:284-303):
    size_bytes,algorithm,chunk_bytes,avg_us,min_us,max_us,iterations."""
    with open(path, "w") as f:
        f.write("size_bytes,algorithm,chunk_bytes,avg_us,min_us,max_us,iterations\n")
        for e in sweep:
            f.write("%d,%s,%d,%.3f,%.3f,%.3f,%d\n" % (e["bytes"], e["algorithm"], e["chunk"], e["ours_mean_us"],
                                                     e["ours_us"]["min"], e["ours_us"]["max"], e["iterations"]))


def bench_params(args, torch, rank, world):
    """BASELINE configs 4/5: broadcast every parameter tensor of a CNN from a
    root (layer-wise, algorithm and chunk tuned per tensor size), per
    iteration, next to NCCL broadcasting the same tensors."""
    import torch.distributed as dist
    import paper_1707_09414_b200 as B
    from paper_1707_09414_b200.comm import DevicePtr
    from paper_1707_09414_b200.params import ParamBroadcaster
    from paper_1707_09414_b200.workloads import MODELS
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    pb = ParamBroadcaster(MODELS[args.workload], bucket_bytes=args.bucket, fused=args.fused)
    comm = B.Comm.connect_torch(world, rank, local, heap_bytes=pb.total_bytes + (16 << 20), timeout_s=30)
    flat = torch.as_tensor(DevicePtr(comm.alloc(pb.total_bytes), pb.total_bytes), device=dev)
    g = torch.Generator(device=dev).manual_seed(2)
    ref = torch.randint(0, 256, (pb.total_bytes,), dtype=torch.uint8, device=dev, generator=g)
    views = [flat[o:o + n] for o, n in pb.msgs]
    stream = torch.cuda.Stream(device=dev)
    nccl_direct = NcclDirect(torch, rank, world)
    torch.cuda.synchronize()
    roots = [0] if args.workload == "vgg16" else [world - 1, world // 2]
    results = {}
    launches_total = 0
    for root in roots:
        for impl in ("ours", "nccl"):
            def prepare(it):
                with torch.cuda.stream(stream):
                    if rank == root:
                        flat.copy_(ref)
                    else:
                        flat.zero_()
                if it == 0:
                    stream.synchronize()
                    dist.barrier(device_ids=[local])

            def issue():
                if impl == "ours":
                    pb.bcast(comm, flat, root, stream)
                else:
                    for v in views:
                        nccl_direct.bcast(v, v.numel(), root, stream)

            graph = None
            per_iter = None
            if args.graph:  # one eager iteration (lazy setup), then capture one
                l_eager = comm.launches
                with torch.cuda.stream(stream):
                    issue()
                per_iter = comm.launches - l_eager  # our kernels per replayed iteration
                stream.synchronize()
                dist.barrier(device_ids=[local])
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph, stream=stream):
                    issue()
                stream.synchronize()
                dist.barrier(device_ids=[local])

            def body(it):
                if graph is None:
                    issue()
                else:
                    with torch.cuda.stream(stream):
                        graph.replay()

            def verify(it):
                return all(torch.equal(flat[o:o + n], ref[o:o + n]) for o, n in zip(pb.offsets, pb.sizes))

            l0 = comm.launches
            # a gate long enough for the host to enqueue every per-tensor call
            # (~10 us of host time each) before the GPU reaches them
            gate = max(GATE_CYCLES, 40_000 * len(pb.msgs))
            times = time_steps(torch, args.steps, args.warmup, prepare, body, verify, stream,
                               align=lambda: comm.barrier(stream), gate=gate)
            if graph is not None:  # destroy it now: NCCL's communicator cannot go while a graph holds its work
                stream.synchronize()
                graph = None
                torch.cuda.synchronize()
            if impl == "ours":  # our kernels in the timed steps (the barrier kernels excluded)
                if per_iter is not None:
                    launches_total += per_iter * args.steps
                else:
                    launches_total += (comm.launches - l0) * args.steps // (args.steps + args.warmup)
            t = torch.tensor(times, dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            results[(root, impl)] = statistics.mean(t.cpu().tolist())
    if rank == 0:
        ours = statistics.mean(results[(r, "ours")] for r in roots)
        nccl = statistics.mean(results[(r, "nccl")] for r in roots)
        line = {"metric": f"{args.workload} layer-wise parameter broadcast time per iteration",
                "value": round(ours * 1e3, 4), "unit": "ms", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ours * 1e3, 4), "higher_is_better": False,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32 (moved as bytes)",
                "data": "synthetic parameters (random bytes), torchvision layer shapes",
                "config": {"workload": f"{args.workload}: {len(pb.sizes)} tensors, {sum(pb.sizes)} bytes, "
                                       f"{len(pb.msgs)} broadcasts per iteration (bucket {args.bucket} B"
                                       f"{', grouped: bcl_group_start/end' if args.fused else ''}"
                                       f"{', CUDA graph replay (ours and NCCL)' if args.graph else ''}), roots {roots}",
                           "tensors": len(pb.sizes), "bytes": sum(pb.sizes), "messages": len(pb.msgs)},
                "per_root_ms": {str(r): {"ours": round(results[(r, 'ours')] * 1e3, 4),
                                         "nccl": round(results[(r, 'nccl')] * 1e3, 4)} for r in roots},
                "nccl_ms": round(nccl * 1e3, 4),
                "link_bound_ms": round(sum(pb.sizes) / LINK_BW * 1e3, 4),
                "gpu_launches": launches_total}
        print(json.dumps(line), flush=True)
    dist.barrier(device_ids=[local])
    nccl_direct.close()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
