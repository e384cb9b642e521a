"""NVLS multicast broadcast (`nvls_kernel`).

The root writes each piece once through the multicast address, the NVSwitch
replicates it into every GPU's copy of the staging ring, receivers copy it
out. Parity: every rank's buffer equals the CPU oracle's (the root payload)
for every schedule the protocol carries, every root, odd sizes, misaligned
buffers, messages that wrap the 64 MiB ring, and back-to-back calls whose
ring counters continue across calls. A multicast team needs two or more
GPUs: on one GPU the tests check that the communicator says so and that the
protocol fails loudly instead of falling back.
"""
import os
import random
import socket

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import _oracle as O  # noqa: E402
import paper_1707_09414_b200 as B  # noqa: E402
from test_multigpu import cfg_of, ngpu, run_group  # noqa: E402

needs2 = pytest.mark.skipif(ngpu() < 2, reason="needs >= 2 GPUs")
needs1 = pytest.mark.skipif(ngpu() < 1, reason="needs a GPU")


def _team(devices, timeout_s=10, **opts):
    comms = B.Comm.local(devices, timeout_s=timeout_s, **opts)
    ok, why = comms[0].nvls()
    if not ok:
        pytest.skip("no multicast team on this box: " + why)
    return comms


@needs1
def test_single_gpu_group_has_no_team_and_nvls_fails_loudly():
    comms = B.Comm.local([0, 0, 0], timeout_s=5)
    ok, why = comms[0].nvls()
    assert not ok and "one GPU" in why
    for c in comms:
        c.set_protocol("nvls")
    bufs = [torch.zeros(4096, dtype=torch.uint8, device="cuda:0") for _ in comms]
    with pytest.raises(ValueError, match="NVLS"):
        B.run_bcast(comms, 0, bufs, 4096, cfg_of("direct"))
    for c in comms:
        c.set_protocol("auto")
    assert comms[0].path(8 << 20, cfg_of("direct")) != "nvls_kernel"
    with pytest.raises(Exception):  # nvls=1 requires the team
        B.Comm.local([0, 0], timeout_s=5, nvls=1)


@needs2
def test_nvls_every_schedule_root_and_size():
    devices = list(range(min(ngpu(), 8)))
    comms = _team(devices)
    for c in comms:
        c.set_protocol("nvls")
    assert comms[0].path(1 << 20, cfg_of("chain_pipelined", 65536)) == "nvls_ll_kernel"  # multicast LL lines
    assert comms[0].path((2 << 20) + 1, cfg_of("chain_pipelined", 65536)) == "nvls_kernel"
    rng = random.Random(41)
    sizes = [1, 15, 16, 17, 4097, (1 << 20) + 3, rng.randrange(1, 9 << 20), (16 << 20) + 5]
    for algo in ("direct", "chain_pipelined", "knomial", "scatter_ring_allgather"):
        for root in range(len(devices)):
            for m in sizes:
                run_group(comms, devices, algo, root, m, chunk=max(1, m // 3 + 1), seed=m * 7 + root)
    # past the 64 MiB ring: pieces wrap the ring inside one call
    run_group(comms, devices, "direct", len(devices) - 1, (150 << 20) + 9, seed=3)
    for c in comms:
        c.set_protocol("auto")


@needs2
def test_nvls_auto_carries_large_direct_and_empty_message():
    devices = list(range(min(ngpu(), 8)))
    comms = _team(devices)
    assert comms[0].path(8 << 20, cfg_of("direct")) == "nvls_kernel"
    assert comms[0].path(1024, cfg_of("direct")) == "ll_kernel/direct"  # LL below its threshold
    assert comms[0].path(8 << 20, cfg_of("chain_pipelined", 1 << 20)) != "nvls_kernel"
    run_group(comms, devices, "direct", 1, (8 << 20) + 1, seed=9)
    run_group(comms, devices, "direct", 0, 0, seed=1)


@needs2
def test_nvls_ll_lines_back_to_back():
    """Multicast LL lines (messages <= 2 MiB): 300 calls back to back, both
    halves of the LL area reused every other call, sizes around the 8-byte
    line payload, misaligned views, rotating roots, every byte checked."""
    devices = list(range(min(ngpu(), 8)))
    n = len(devices)
    comms = _team(devices)
    for c in comms:
        c.set_protocol("nvls")
    rng = random.Random(97)
    cap = 2 << 20
    bufs = [torch.empty(cap + 16, dtype=torch.uint8, device=f"cuda:{d}") for d in devices]
    try:
        for it in range(300):
            m = rng.choice([1, 7, 8, 9, 4095, rng.randrange(1, 70000), rng.randrange(70000, cap + 1), cap])
            off = rng.randrange(0, 9)
            root = (it * 5) % n
            src = torch.randint(0, 256, (m,), dtype=torch.uint8, device=f"cuda:{devices[root]}")
            views = [b[off:off + m] for b in bufs]
            for r in range(n):
                (views[r].copy_(src) if r == root else views[r].fill_(it & 0xFF))
            torch.cuda.synchronize(devices[root])
            assert comms[0].path(m, cfg_of("direct")) == "nvls_ll_kernel"
            B.run_bcast(comms, root, views, m, cfg_of("direct"))
            for r in range(n):
                assert torch.equal(views[r].cpu(), src.cpu()), (it, m, off, root, r)
    finally:
        for c in comms:
            c.set_protocol("auto")


@needs2
def test_nvls_misaligned_buffers():
    devices = list(range(min(ngpu(), 8)))
    n = len(devices)
    comms = _team(devices)
    for c in comms:
        c.set_protocol("nvls")
    base = [torch.empty((4 << 20) + 64, dtype=torch.uint8, device=f"cuda:{d}") for d in devices]
    for it, (m, offs) in enumerate([((1 << 20) + 3, [1, 2, 3, 5]), (12345, [7, 0, 4, 1]), ((3 << 20) + 1, [0, 9, 0, 13])]):
        root = it % n
        src = torch.randint(0, 256, (m,), dtype=torch.uint8, device=f"cuda:{devices[root]}")
        views = [base[r][offs[r % 4]:offs[r % 4] + m] for r in range(n)]
        for r in range(n):
            (views[r].copy_(src) if r == root else views[r].fill_(0x5A))
        torch.cuda.synchronize(devices[root])
        B.run_bcast(comms, root, views, m, cfg_of("direct"))
        for r in range(n):
            assert torch.equal(views[r].cpu(), src.cpu()), (m, offs, r)
    for c in comms:
        c.set_protocol("auto")


@needs2
@pytest.mark.parametrize("strict", [0, 1])
def test_nvls_back_to_back_stress(strict):
    """Monotone ring counters across calls: 200 calls back to back (sizes from
    one piece to several ring wraps' worth of slots), fresh payloads, rotating
    roots, every byte checked before the next call."""
    devices = list(range(min(ngpu(), 8)))
    n = len(devices)
    comms = _team(devices, nvls_strict=strict)
    for c in comms:
        c.set_protocol("nvls")
    rng = random.Random(53 + strict)
    cap = 24 << 20
    bufs = [torch.empty(cap, dtype=torch.uint8, device=f"cuda:{d}") for d in devices]
    try:
        for it in range(200):
            m = rng.choice([rng.randrange(1, 70000), rng.randrange(70000, 4 << 20), rng.randrange(4 << 20, cap + 1)])
            root = (it * 3) % n
            src = torch.randint(0, 256, (m,), dtype=torch.uint8, device=f"cuda:{devices[root]}")
            for r in range(n):
                (bufs[r][:m].copy_(src) if r == root else bufs[r][:m].fill_((it * 5) & 0xFF))
            torch.cuda.synchronize(devices[root])
            B.run_bcast(comms, root, [b[:m] for b in bufs], m, cfg_of("direct"))
            for r in range(n):
                assert torch.equal(bufs[r][:m].cpu(), src.cpu()), (it, m, root, r)
    finally:
        for c in comms:
            c.set_protocol("auto")


@needs2
def test_nvls_ranks_sharing_gpus():
    devices = [d for d in range(min(ngpu(), 4)) for _ in range(2)]
    comms = _team(devices)
    for c in comms:
        c.set_protocol("nvls")
    for root in (0, len(devices) - 1, len(devices) // 2 + 1):
        run_group(comms, devices, "direct", root, (5 << 20) + 11, seed=root)
    for c in comms:
        c.set_protocol("auto")


@needs2
def test_nvls_missing_root_times_out_with_named_error():
    comms = _team([0, 1], timeout_s=1.0)
    comms[0].set_protocol("nvls")
    buf = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda:0")
    comms[0].bcast(buf, 1 << 20, "uint8", 1, cfg_of("direct"))  # the root (rank 1) never calls
    with pytest.raises(B.DeviceTimeout) as e:
        comms[0].check()
    assert "rank 0" in str(e.value)


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
        comm = B.Comm.connect_torch(world, rank, rank, heap_bytes=0, timeout_s=10)
        ok, why = comm.nvls()
        if not ok:
            q.put((rank, None, why))
            return
        comm.set_protocol("nvls")
        # arbitrary torch buffers, no registration: peers never touch them
        plain = torch.zeros((80 << 20) + 64, dtype=torch.uint8, device=f"cuda:{rank}")
        good = True
        for it, (m, root, off) in enumerate([(64 << 20, 0, 0), (12345, world - 1, 3), ((70 << 20) + 1, 1 % world, 1),
                                             (1, 0, 0), ((3 << 20) + 5, world - 1, 16)]):
            payload = O.payload(500 + it, m)
            view = plain[off:off + m]
            (view.copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8)) if rank == root else view.zero_())
            torch.cuda.synchronize()
            dist.barrier()
            comm.bcast(view, m, "uint8", root, cfg_of("direct"))
            comm.check()
            good &= view.cpu().numpy().tobytes() == payload
        q.put((rank, good, comm.path(64 << 20, cfg_of("direct"))))
        comm.close()
    except Exception as e:  # noqa: BLE001
        q.put((rank, False, repr(e)))
    finally:
        dist.destroy_process_group()


@needs2
def test_nvls_one_process_per_gpu():
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
    if all(ok is None for _, ok, _ in res):
        pytest.skip("no multicast team across processes: " + res[0][2])
    for rank, ok, info in res:
        assert ok, res
        assert info == "nvls_kernel"
