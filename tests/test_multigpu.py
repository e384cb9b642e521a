"""Multi-GPU parity (needs >= 2 visible B200s; skipped otherwise).

* one process driving every GPU (UVA + peer access): all algorithms, roots;
* 2 ranks per GPU on the available GPUs (8 ranks on 4 GPUs);
* one process per GPU over CUDA IPC (the bench.py shape), spawned here with
  a gloo rendezvous for the handle exchange;
* a rank that never joins makes its peers time out with a named error.
"""
import os
import random
import socket

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import _oracle as O  # noqa: E402
import paper_1707_09414_b200 as B  # noqa: E402


def ngpu():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


needs2 = pytest.mark.skipif(ngpu() < 2, reason="needs >= 2 GPUs")


def cfg_of(algo, chunk=0, radix=0):
    a = B.Algorithm[algo]
    return B.AlgorithmConfig(a, radix if a in (B.Algorithm.knomial, B.Algorithm.knomial_staged) else 0,
                             chunk if a == B.Algorithm.chain_pipelined else 0)


def run_group(comms, devices, algo, root, m, chunk=0, radix=2, seed=1):
    n = len(devices)
    payload = O.payload(seed, m)
    expect = [bytearray(m) for _ in range(n)]
    expect[root][:] = payload
    O.bcast(algo, n, root, expect, chunk=chunk, radix=radix)
    bufs = [torch.zeros(m, dtype=torch.uint8, device=f"cuda:{d}") for d in devices]
    if m:
        bufs[root].copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8))
    B.run_bcast(comms, root, bufs, m, cfg_of(algo, chunk, radix))
    for r in range(n):
        assert bufs[r].cpu().numpy().tobytes() == bytes(expect[r]), (algo, n, root, m, chunk, r)


@needs2
def test_one_process_all_gpus_every_algorithm_and_root():
    devices = list(range(min(ngpu(), 8)))
    comms = B.Comm.local(devices, timeout_s=10)
    assert comms[0].protocol_caps()["ll128"] == 1 << 62  # own GPU each: LL128 ring, no size limit but the table rule
    rng = random.Random(17)
    for algo in ("chain_pipelined", "chain_pipelined/ll", "chain_pipelined/pull", "chain_pipelined/push",
                 "knomial", "scatter_ring_allgather", "direct", "chain"):
        algo, _, protocol = algo.partition("/")
        for c in comms:
            c.set_protocol(protocol or "auto")  # auto: LL128 lines up to 32 MiB; pull: the lane executor
        for root in range(len(devices)):
            big = (8 << 20) - 3 if protocol == "ll" else (8 << 20) + 5  # the LL chain cap is 8 MiB
            for m in (0, 4, 4097, 1 << 20, rng.randrange(1, 5 << 20), big):
                run_group(comms, devices, algo, root, m, chunk=max(1, m // 5 + 3), seed=m + root)
    for protocol in ("push", "auto"):  # full size on the producer-store path too
        for c in comms:
            c.set_protocol(protocol)
        run_group(comms, devices, "chain_pipelined", 0, 64 << 20, chunk=512 << 10, seed=5)


@needs2
def test_ll128_chain_back_to_back_stress():
    """LL128 relies on 128-byte NVLink stores arriving whole: many calls back
    to back with fresh payloads, every size class, roots rotating, every
    result checked before the next call reuses the landing halves."""
    devices = list(range(min(ngpu(), 8)))
    n = len(devices)
    old = os.environ.get("BCL_LL128_MAX")
    os.environ["BCL_LL128_MAX"] = str(32 << 20)
    try:
        comms = B.Comm.local(devices, timeout_s=10)
    finally:
        if old is None:
            os.environ.pop("BCL_LL128_MAX")
        else:
            os.environ["BCL_LL128_MAX"] = old
    for c in comms:
        c.set_protocol("ll128")
    rng = random.Random(23)
    cap = 32 << 20
    bufs = [torch.empty(cap + 64, dtype=torch.uint8, device=f"cuda:{d}") for d in devices]
    sizes = [1, 119, 120, 121, 4096, 1 << 20, (1 << 20) + 7, 5 << 20, cap - 1, cap]
    for it in range(60):
        m = sizes[it % len(sizes)] if it < 2 * len(sizes) else rng.randrange(1, cap + 1)
        root = it % n
        src = torch.randint(0, 256, (m,), dtype=torch.uint8, device=f"cuda:{devices[root]}")
        for r in range(n):
            if r == root:
                bufs[r][:m].copy_(src)
            else:
                bufs[r][:m].fill_(it & 0xFF)
        torch.cuda.synchronize(devices[root])
        B.run_bcast(comms, root, [b[:m] for b in bufs], m, cfg_of("chain_pipelined", 262144))
        for r in range(n):
            assert torch.equal(bufs[r][:m].cpu(), src.cpu()), (it, m, root, r)
    # misaligned buffers (byte paths of the 120-byte payload pieces)
    for it, (m, offs) in enumerate([((1 << 20) + 3, [1, 2, 3, 5]), (12345, [7, 0, 4, 1]), (120 * 1000 + 1, [3, 3, 3, 3])]):
        root = it % n
        src = torch.randint(0, 256, (m,), dtype=torch.uint8, device=f"cuda:{devices[root]}")
        views = [bufs[r][offs[r % 4]:offs[r % 4] + m] for r in range(n)]
        for r in range(n):
            (views[r].copy_(src) if r == root else views[r].fill_(0xA5))
        torch.cuda.synchronize(devices[root])
        B.run_bcast(comms, root, views, m, cfg_of("chain_pipelined", 262144))
        for r in range(n):
            assert torch.equal(views[r].cpu(), src.cpu()), ("misaligned", m, offs, r)
    with pytest.raises(ValueError):  # above the communicator's ll128_max
        B.run_bcast(comms, 0, [b[:cap + 1] for b in bufs], cap + 1, cfg_of("chain_pipelined", 262144))
    for c in comms:
        c.set_protocol("auto")


@needs2
def test_ll128_direct_lines():
    """`direct` calls from ll128_direct_min up to the LL threshold travel as
    128-byte LL128 lines (their own landing areas, the LL direct halves and
    credits): sizes around both thresholds and the 120-byte line payload,
    every root, misaligned views, the two formats interleaved back to back on
    the same halves (each result checked before the next call), a grouped run
    (fused LL128 direct lines with the small members as segments)."""
    devices = list(range(min(ngpu(), 8)))
    n = len(devices)
    comms = B.Comm.local(devices, timeout_s=10, ll128_direct_min=65536)
    d = cfg_of("direct")
    ll_max = comms[0].protocol_caps()["ll_direct"]
    assert comms[0].path(65535, d) == "ll_kernel/direct"
    assert comms[0].path(65536, d) == comms[0].path(ll_max, d) == "ll128_kernel/direct"
    assert comms[0].path(ll_max + 1, d) != "ll128_kernel/direct"
    for root in range(n):
        for m in (65535, 65536, 65537, 120 * 600, 120 * 600 + 1, 1 << 20, ll_max - 1, ll_max, ll_max + 1):
            run_group(comms, devices, "direct", root, m, seed=m + root)
    rng = random.Random(29)
    cap = ll_max + 64
    bufs = [torch.empty(cap, dtype=torch.uint8, device=f"cuda:{x}") for x in devices]
    for it in range(80):
        m = rng.choice([rng.randrange(1, 65536), rng.randrange(65536, ll_max + 1)])
        off = rng.randrange(0, 16) if it % 3 == 0 else 0
        root = rng.randrange(n)
        src = torch.randint(0, 256, (m,), dtype=torch.uint8, device=f"cuda:{devices[root]}")
        views = [b[off:off + m] for b in bufs]
        for r in range(n):
            (views[r].copy_(src) if r == root else views[r].fill_(it & 0xFF))
        torch.cuda.synchronize(devices[root])
        B.run_bcast(comms, root, views, m, d)
        for r in range(n):
            assert torch.equal(views[r].cpu(), src.cpu()), (it, m, off, root, r)
    sizes = [5000, 300000, 777, 70000, 40000, 2 << 20 if ll_max >= 2 << 20 else ll_max]
    views, srcs, at = [], [], 0
    for k, m in enumerate(sizes):
        views.append([b[at:at + m] for b in bufs] if at + m <= cap else None)
        at += m
    views = [v for v in views if v is not None]
    streams = [torch.cuda.Stream(device=f"cuda:{x}") for x in devices]
    for k, v in enumerate(views):
        src = torch.randint(0, 256, (v[0].numel(),), dtype=torch.uint8, device=f"cuda:{devices[k % n]}")
        for r in range(n):
            (v[r].copy_(src) if r == k % n else v[r].zero_())
        srcs.append(src)
    for x in devices:
        torch.cuda.synchronize(x)
    with B.group():
        for k, v in enumerate(views):
            B.bcast_all(comms, v, v[0].numel(), "uint8", k % n, d, streams=streams)
    for x in devices:
        torch.cuda.synchronize(x)
    for k, (v, src) in enumerate(zip(views, srcs)):
        for r in range(n):
            assert torch.equal(v[r].cpu(), src.cpu()), ("group", k, r)
    for c in comms:
        c.check()
    off = B.Comm.local(devices, timeout_s=10, ll128_direct_min=0)
    assert off[0].path(1 << 20, d) == "ll_kernel/direct"
    run_group(off, devices, "direct", n - 1, (1 << 20) + 3, seed=3)


@needs2
def test_pull_flag_ordering_litmus():
    """The default pull path publishes a slice after a gpu-scope fence of the
    producing warp (DESIGN.md §5 "Memory ordering": the producer's L2 is the
    point of coherence for NVLink readers, a hardware property rather than a
    PTX-model guarantee). Litmus-style stress: 300 back-to-back broadcasts
    with small chunks and slices (thousands of flag hand-offs per call), a
    fresh payload and a rotating root every call, every byte of every rank
    checked before the next call reuses the buffers."""
    devices = list(range(min(ngpu(), 8)))
    n = len(devices)
    comms = B.Comm.local(devices, timeout_s=10, min_slice=512, window_bytes=1 << 20)
    for c in comms:
        c.set_protocol("pull")
    rng = random.Random(31)
    cap = 4 << 20
    bufs = [torch.empty(cap, dtype=torch.uint8, device=f"cuda:{d}") for d in devices]
    try:
        for it in range(300):
            m = rng.choice([rng.randrange(1, 65536), rng.randrange(65536, cap), cap])
            chunk = rng.choice([4096, 8192, 16384, 65536])
            root = it % n
            src = torch.randint(0, 256, (m,), dtype=torch.uint8, device=f"cuda:{devices[root]}")
            for r in range(n):
                (bufs[r][:m].copy_(src) if r == root else bufs[r][:m].fill_((it * 7) & 0xFF))
            torch.cuda.synchronize(devices[root])
            B.run_bcast(comms, root, [b[:m] for b in bufs], m, cfg_of("chain_pipelined", chunk))
            for r in range(n):
                assert torch.equal(bufs[r][:m].cpu(), src.cpu()), (it, m, chunk, root, r)
    finally:
        for c in comms:
            c.set_protocol("auto")


@needs2
def test_two_ranks_per_gpu():
    devices = [d for d in range(min(ngpu(), 4)) for _ in range(2)]
    comms = B.Comm.local(devices, timeout_s=10)
    for algo in ("chain_pipelined", "scatter_ring_allgather", "knomial"):
        for root in (0, len(devices) - 1, len(devices) // 2):
            run_group(comms, devices, algo, root, (3 << 20) + 5, chunk=262147, seed=root)


@needs2
def test_missing_rank_times_out_with_named_error():
    comms = B.Comm.local([0, 1], timeout_s=1.0)
    buf = torch.zeros(4096, dtype=torch.uint8, device="cuda:0")
    comms[0].bcast(buf, 4096, "uint8", 1, cfg_of("chain_pipelined", 1024))  # rank 1 never calls
    with pytest.raises(B.DeviceTimeout) as e:
        comms[0].check()
    assert "rank 0" in str(e.value) and "peer 1" in str(e.value)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(rank)
        from paper_1707_09414_b200.comm import DevicePtr
        comm = B.Comm.connect_torch(world, rank, rank, heap_bytes=96 << 20, timeout_s=10)
        cap = 70 << 20
        buf = torch.as_tensor(DevicePtr(comm.alloc(cap), cap), device=f"cuda:{rank}")
        ok = True
        for it, (algo, m, root) in enumerate([("chain_pipelined", 64 << 20, 0), ("knomial", 12345, world - 1),
                                              ("scatter_ring_allgather", 3 << 20, 1 % world),
                                              ("chain_pipelined", 1, 0), ("direct", 777, 0),
                                              ("chain_pipelined", (5 << 20) + 3, world - 1),
                                              ("chain_pipelined", 8 << 20, 1 % world),
                                              ("direct", 1 << 20, world - 1),
                                              ("direct", 2 << 20, 0), ("direct", (128 << 10) + 5, 1 % world),
                                              ("chain_pipelined", (3 << 20) + 1, 0)]):
            payload = O.payload(it, m)
            if rank == root:
                buf[:m].copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8))
            else:
                buf[:m].zero_()
            torch.cuda.synchronize()
            dist.barrier()
            comm.bcast(buf, m, "uint8", root, cfg_of(algo, 524288, 2))
            comm.check()
            ok &= buf[:m].cpu().numpy().tobytes() == payload
        # arbitrary cudaMalloc'd buffers (torch's allocator): the line
        # protocols take them as they are; the lane executor after a
        # collective registration of their allocation (bcl_comm_register_*)
        plain = torch.zeros((6 << 20) + 64, dtype=torch.uint8, device=f"cuda:{rank}")
        for it, (proto, m, root, off) in enumerate([("auto", 100000, 0, 0), ("ll128", (5 << 20) + 1, world - 1, 3)]):
            comm.set_protocol(proto)
            payload = O.payload(200 + it, m)
            view = plain[off:off + m]
            (view.copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8)) if rank == root else view.zero_())
            torch.cuda.synchronize()
            dist.barrier()
            comm.bcast(view, m, "uint8", root, cfg_of("chain_pipelined", 65536))
            comm.check()
            ok &= view.cpu().numpy().tobytes() == payload
        comm.register(plain)
        for it, (proto, m, root, off) in enumerate([("pull", (6 << 20) + 7, 0, 5), ("push", 1 << 20, world - 1, 0),
                                                    ("pull", 3 << 20, 1 % world, 16)]):
            comm.set_protocol(proto)
            payload = O.payload(300 + it, m)
            view = plain[off:off + m]
            (view.copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8)) if rank == root else view.zero_())
            torch.cuda.synchronize()
            dist.barrier()
            comm.bcast(view, m, "uint8", root, cfg_of("chain_pipelined", 262144))
            comm.check()
            ok &= view.cpu().numpy().tobytes() == payload
        comm.set_protocol("auto")
        # grouped per-rank calls (bcl_group_start/end): every rank fuses alike
        msgs = [(1, 0), (300, 64), (70000, 1024), ((2 << 20) + 5, 80000), (17, (3 << 20)), ((1 << 20) + 3, 4 << 20)]
        payloads = []
        root = world - 1
        for k, (m, off) in enumerate(msgs):
            payload = O.payload(400 + k, m)
            view = plain[off:off + m]
            (view.copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8)) if rank == root else view.zero_())
            payloads.append(payload)
        torch.cuda.synchronize()
        dist.barrier()
        before = comm.launches
        with B.group():
            for m, off in msgs:
                comm.bcast(plain[off:off + m], m, "uint8", root, None)
        comm.check()
        ok &= comm.launches - before < len(msgs)
        for (m, off), payload in zip(msgs, payloads):
            ok &= plain[off:off + m].cpu().numpy().tobytes() == payload
        # host-buffer entry point (pipelined H2D / broadcast / D2H pieces)
        m = (9 << 20) + 3
        payload = O.payload(99, m)
        host = torch.zeros(m, dtype=torch.uint8).pin_memory()
        if rank == 1 % world:
            host.copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8))
        dist.barrier()
        comm.bcast_host(host, m, "uint8", 1 % world, cfg_of("chain_pipelined", 262144))
        comm.check()
        ok &= host.numpy().tobytes() == payload
        q.put((rank, ok, None))
        comm.close()
    except Exception as e:  # noqa: BLE001
        q.put((rank, False, repr(e)))
    finally:
        dist.destroy_process_group()


@needs2
def test_one_process_per_gpu_over_ipc():
    import torch.multiprocessing as mp
    world = min(ngpu(), 4)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank, ok, err in res:
        assert ok, (rank, err)


@needs2
def test_group_fusion_across_gpus():
    """bcl_group_start/end across GPUs: runs of LL128 chain calls and of LL
    direct calls fuse into shared launches (odd sizes, every root), calls on
    the lane executor stay separate, everything bit-exact and in order."""
    devices = list(range(min(ngpu(), 8)))
    n = len(devices)
    comms = B.Comm.local(devices, timeout_s=10)
    rng = random.Random(83)
    for root in range(n):
        sizes = [rng.choice([1, 119, 120, 121, 5000, rng.randrange(1, 3 << 20)]) for _ in range(12)]
        algos = ["chain_pipelined"] * 6 + ["direct"] * 5 + ["chain_pipelined"]
        bufs = [[torch.empty(m, dtype=torch.uint8, device=f"cuda:{d}") for d in devices] for m in sizes]
        srcs = []
        for k, m in enumerate(sizes):
            src = torch.randint(0, 256, (m,), dtype=torch.uint8, device=f"cuda:{devices[root]}")
            for r in range(n):
                (bufs[k][r].copy_(src) if r == root else bufs[k][r].fill_(0x77))
            srcs.append(src)
        for d in devices:
            torch.cuda.synchronize(d)
        before = comms[0].launches
        with B.group():
            for k, m in enumerate(sizes):
                B.bcast_all(comms, bufs[k], m, "uint8", root, cfg_of(algos[k], 262144))
        for d in devices:
            torch.cuda.synchronize(d)
        assert comms[0].launches - before <= 3, comms[0].launches - before
        for k in range(len(sizes)):
            for r in range(n):
                assert torch.equal(bufs[k][r].cpu(), srcs[k].cpu()), (root, k, sizes[k], r)
    # a large chain call inside the group goes to the lane executor, alone
    big = [torch.zeros(64 << 20, dtype=torch.uint8, device=f"cuda:{d}") for d in devices]
    big[0].fill_(9)
    small = [torch.zeros(999, dtype=torch.uint8, device=f"cuda:{d}") for d in devices]
    small[0].fill_(5)
    for c in comms:
        c.set_protocol("pull")
    try:
        with B.group():
            B.bcast_all(comms, small, 999, "uint8", 0, cfg_of("direct"))
            B.bcast_all(comms, big, 64 << 20, "uint8", 0, cfg_of("chain_pipelined", 65536))
            B.bcast_all(comms, small, 999, "uint8", 0, cfg_of("direct"))
    finally:
        for c in comms:
            c.set_protocol("auto")
    for d in devices:
        torch.cuda.synchronize(d)
    for r in range(n):
        assert int(big[r].min()) == 9 == int(big[r].max()) and int(small[r].min()) == 5 == int(small[r].max())


@needs2
def test_one_gibibyte_across_gpus_every_transport():
    """1 GiB (the sweep's top size) across GPUs on the default transport
    (LL128 from n = 3, pull at n = 2) and on push; every byte checked."""
    devices = list(range(min(ngpu(), 4)))
    n, m = len(devices), 1 << 30
    comms = B.Comm.local(devices, timeout_s=20)
    bufs = [torch.zeros(m, dtype=torch.uint8, device=f"cuda:{d}") for d in devices]
    g = torch.Generator(device=f"cuda:{devices[-1]}").manual_seed(5)
    src = torch.randint(0, 256, (m,), dtype=torch.uint8, device=f"cuda:{devices[-1]}", generator=g)
    for proto in ("auto", "push"):
        for c in comms:
            c.set_protocol(proto)
        for r in range(n):
            (bufs[r].copy_(src) if r == n - 1 else bufs[r].zero_())
        for d in devices:
            torch.cuda.synchronize(d)
        B.run_bcast(comms, n - 1, bufs, m, cfg_of("chain_pipelined", 1 << 20))
        for r in range(n):
            assert torch.equal(bufs[r], src.to(f"cuda:{devices[r]}")), (proto, r)
    for c in comms:
        c.set_protocol("auto")


@needs2
@pytest.mark.parametrize("proto", ["auto", "pull", "push", "nvls"])
def test_graph_capture_replays_across_gpus(proto):
    """Captured broadcasts across GPUs (LL128 / pull / push / NVLS): the
    device-side call state gives every replay a fresh epoch and ring
    position; 5 replays with fresh payloads, every byte checked."""
    devices = list(range(min(ngpu(), 4)))
    n = len(devices)
    comms = B.Comm.local(devices, timeout_s=10)
    if proto == "nvls" and not comms[0].nvls()[0]:
        pytest.skip("no multicast team")
    for c in comms:
        c.set_protocol(proto)
    sizes = [(8 << 20) + 5, 3000, (1 << 20) + 9]  # the last one on the `direct` schedule (LL128 direct lines)
    bufs = [[torch.zeros(m, dtype=torch.uint8, device=f"cuda:{d}") for d in devices] for m in sizes]
    streams = [torch.cuda.Stream(device=f"cuda:{d}") for d in devices]

    def body():
        for k, m in enumerate(sizes):
            cfg = cfg_of("direct") if k == 2 else cfg_of("chain_pipelined", 262144)
            B.bcast_all(comms, bufs[k], m, "uint8", (k + 1) % n, cfg, streams=streams)

    body()  # warm-up outside capture
    for d in devices:
        torch.cuda.synchronize(d)
    # one process, several GPUs: capture every GPU's stream into one graph
    # (the other streams join the capturing stream through events)
    g = torch.cuda.CUDAGraph()
    cap = streams[0]
    ev = [torch.cuda.Event() for _ in devices]
    with torch.cuda.graph(g, stream=cap):
        start = torch.cuda.Event()
        start.record(cap)
        for i, st in enumerate(streams[1:], 1):
            st.wait_event(start)
        body()
        for i, st in enumerate(streams[1:], 1):
            ev[i].record(st)
            cap.wait_event(ev[i])
    for d in devices:
        torch.cuda.synchronize(d)
    try:
        for rep in range(5):
            vals = [(rep * 2 + k) % 250 + 3 for k in range(len(sizes))]
            for k in range(len(sizes)):
                for r in range(n):
                    bufs[k][r].fill_(vals[k] if r == (k + 1) % n else 0)
            for d in devices:
                torch.cuda.synchronize(d)
            with torch.cuda.stream(cap):
                g.replay()
            for d in devices:
                torch.cuda.synchronize(d)
            for k in range(len(sizes)):
                for r in range(n):
                    assert int(bufs[k][r].min()) == vals[k] == int(bufs[k][r].max()), (proto, rep, k, r)
        for c in comms:
            c.check()
    finally:
        for c in comms:
            c.set_protocol("auto")


@needs2
def test_soak_every_transport_groups_and_graphs():
    """tools/r2/soak.py, short: random calls across every transport, schedule,
    root and size, grouped runs, barriers and a replayed CUDA graph, every
    byte checked after each step."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "tools", "r2", "soak.py"), "150", "11"],
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0 and "soak ok" in out.stdout, out.stdout[-2000:] + out.stderr[-2000:]
