"""GPU parity: the device broadcast vs the CPU oracle, bit-exact.

All ranks share cuda:0 here (one cooperative launch serves them). Communicator
options force the cross-GPU device paths onto this one GPU, so every one of
them is checked here (VARIANTS): TMA-bulk pulls with system-scope flags and
writer fences (the default across GPUs), the strict fence mode, producer
pushes, and LL128 lines; tests/test_multigpu.py repeats the key cases across
real GPUs. Cases follow
the reference's own tests: acceptance criterion 4's random trials
(proj/tests/acceptance.cpp:190-233) via the committed golden list, the
runtime tests (proj/tests/test_runtime.cpp:99-254) and edge cases (empty,
ragged, misaligned, C not dividing M, every root).
"""
import json
import os
import random

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import _oracle as O  # noqa: E402
import paper_1707_09414_b200 as B  # noqa: E402

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield
    torch.cuda.synchronize()


_GROUPS = {}

# Device paths of the pipelined chain, as (group options, protocol):
#   auto       the fused per-item kernel auto mode picks on one GPU
#   pull       the lane executor with 16-byte vector loads, gpu-scope flags
#   ll         16-byte LL lines forwarded hop by hop
#   push       producers store into the downstream buffer
#   xpull      what runs across GPUs: TMA bulk pulls through shared-memory
#              stages, system-scope polls and writer fences (chain_pull_bulk)
#   xstrict    the same with the publisher's system-scope fence per flag batch
#   xpush      TMA bulk pushes with system-scope publication
#   ll128      128-byte LL128 lines (the cross-GPU kernel, here through L2)
XGPU = {"stage_bytes": 8192, "sys_scope": 1}
VARIANTS = {
    "auto": ({}, "auto"),
    "pull": ({}, "pull"),
    "ll": ({}, "ll"),
    "push": ({}, "push"),
    "xpull": (dict(XGPU, strict_sys=0), "pull"),  # gpu-scope writer fence (opt-in)
    "xstrict": (XGPU, "pull"),                   # system-scope publisher release (default)
    "xpush": (XGPU, "push"),
    "ll128": ({"ll128": 1, "ll128_max": 32 << 20, "sys_scope": 1}, "ll128"),
}
CHAIN_PROTOCOLS = list(VARIANTS)


def comms_for(n, options=None):
    """One emulated group per (rank count, options), reused across tests (epochs advance)."""
    key = (n, tuple(sorted((options or {}).items())))
    if key not in _GROUPS:
        _GROUPS[key] = B.Comm.local([0] * n, timeout_s=10, **(options or {}))
    return _GROUPS[key]


def cfg_of(algo, chunk=0, radix=0):
    a = B.Algorithm[algo]
    return B.AlgorithmConfig(a, radix if a in (B.Algorithm.knomial, B.Algorithm.knomial_staged) else 0,
                             chunk if a == B.Algorithm.chain_pipelined else 0)


def make_bufs(n, m, root, payload, offsets=None):
    """Device buffers (optionally at byte offsets into larger allocations)."""
    offsets = offsets or [0] * n
    store = [torch.zeros(m + 64, dtype=torch.uint8, device="cuda:0") for _ in range(n)]
    views = [store[r][offsets[r]:offsets[r] + m] for r in range(n)]
    if m:
        views[root].copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8))
    return store, views


def run_case(algo, n, root, m, chunk=0, radix=0, seed=1, offsets=None, protocol="auto"):
    """protocol: a key of VARIANTS (the chain's device path; other schedules
    run on the lane executor with the variant's options)."""
    options, proto = VARIANTS[protocol]
    payload = O.payload(seed, m)
    expect = [bytearray(m) for _ in range(n)]
    expect[root][:] = payload
    O.bcast(algo, n, root, expect, chunk=chunk, radix=radix)
    _, views = make_bufs(n, m, root, payload, offsets)
    comms = comms_for(n, options)
    for c in comms:
        c.set_protocol(proto if algo == "chain_pipelined" else "auto")
    try:
        B.run_bcast(comms, root, views, m, cfg_of(algo, chunk, radix))
    finally:
        for c in comms:
            c.set_protocol("auto")
    for r in range(n):
        got = views[r].cpu().numpy().tobytes()
        assert got == bytes(expect[r]), f"{algo}/{protocol} n={n} root={root} M={m} C={chunk}: rank {r} differs"


@pytest.mark.parametrize("idx", range(len(GOLD["bcasts"])))
def test_reference_trials_bit_exact(idx):
    """Every golden trial: device result == reference result (FNV per rank)."""
    algo, n, root, m, chunk, radix, seed = GOLD["bcasts"][idx]["case"]
    if algo == "chain_pipelined" and n < 2:
        pytest.skip("n < 2")
    payload = O.payload(seed, m)
    _, views = make_bufs(n, m, root, payload)
    B.run_bcast(comms_for(n), root, views, m, cfg_of(algo, chunk, radix))
    got = ["%016x" % O.fnv(views[r].cpu().numpy().tobytes()) for r in range(n)]
    assert got == GOLD["bcasts"][idx]["rank_fnv"]


@pytest.mark.parametrize("algo", ["direct", "chain", "knomial", "scatter_ring_allgather", "knomial_staged",
                                  "direct/xpull", "knomial/xpull", "scatter_ring_allgather/xpull"]
                         + ["chain_pipelined/" + v for v in VARIANTS])
@pytest.mark.parametrize("m", [0, 1, 4, 15, 16, 17, 1000, 4096, 65537])
def test_every_root_small_sizes(algo, m):
    algo, _, protocol = algo.partition("/")
    for n in (2, 3, 5, 8):
        for root in range(n):
            run_case(algo, n, root, m, chunk=max(1, m // 3 + 1) if m else 7, radix=2 + root % 3,
                     seed=m * 31 + root, protocol=protocol or "auto")


@pytest.mark.parametrize("protocol", CHAIN_PROTOCOLS)
def test_chunk_not_dividing_message_and_tiny_chunks(protocol):
    # C in [1, M+1] as acceptance.cpp:203-205 draws it.
    rng = random.Random(5)
    for _ in range(20):
        n = rng.randrange(2, 9)
        m = rng.randrange(0, 300000)
        chunk = 1 + rng.randrange(m + 1)
        if (m + chunk - 1) // max(chunk, 1) > 200000:
            chunk = m // 200000 + 1
        run_case("chain_pipelined", n, rng.randrange(n), m, chunk=chunk, seed=rng.randrange(1 << 30),
                 protocol=protocol)


@pytest.mark.parametrize("protocol", CHAIN_PROTOCOLS)
def test_misaligned_buffers(protocol):
    """Different byte misalignments per rank (vector and byte paths)."""
    for offs in ([0, 1, 2, 3], [5, 5, 5, 5], [16, 3, 0, 9]):
        for algo in ("chain_pipelined", "knomial", "scatter_ring_allgather"):
            run_case(algo, 4, 1, 100003, chunk=8191, radix=2, seed=11, offsets=offs, protocol=protocol)


@pytest.mark.parametrize("protocol", CHAIN_PROTOCOLS)
def test_sixteen_ranks_one_megabyte(protocol):
    # proj/tests/test_runtime.cpp:224-236 shape.
    run_case("chain_pipelined", 16, 0, 1 << 20, chunk=65536, seed=99, protocol=protocol)
    run_case("scatter_ring_allgather", 16, 5, 1 << 20, seed=98)


def test_ll_chain_cap_and_interleaving_with_direct():
    """LL chain at and around its cap (8 MiB), interleaved with LL direct
    calls from changing roots: direct and chain calls keep separate credits
    and landing halves; above the cap the auto path takes over."""
    n = 4
    cap = 8 << 20
    sizes = [cap, cap - 8, 3 << 20, cap + 16, 100, 2 << 20]
    for i, m in enumerate(sizes * 2):
        root = (i * 3) % n
        if i % 2:
            run_case("direct", n, root, m, seed=i + 7)
        else:
            run_case("chain_pipelined", n, root, m, chunk=262144, seed=i + 7,
                     protocol="ll" if m <= cap else "auto")
    with pytest.raises(ValueError):
        run_case("chain_pipelined", n, 0, cap + 16, chunk=262144, protocol="ll")


def test_config1_full_size_all_ranks_equal_root():
    """BASELINE config 1 at full size: 4 ranks, 64 MiB, 512 KiB chunks."""
    n, m, chunk = 4, 64 << 20, 512 << 10
    g = torch.Generator(device="cuda:0").manual_seed(1)
    bufs = [torch.zeros(m, dtype=torch.uint8, device="cuda:0") for _ in range(n)]
    bufs[0].copy_(torch.randint(0, 256, (m,), dtype=torch.uint8, device="cuda:0", generator=g))
    B.run_bcast(comms_for(n), 0, bufs, m, cfg_of("chain_pipelined", chunk))
    for r in range(1, n):
        assert torch.equal(bufs[r], bufs[0])


@pytest.mark.parametrize("root,chunk", [(0, 4 << 20), (3, 65536)])
def test_one_gibibyte_every_rank_equals_root(root, chunk):
    """The sweep's largest size (BASELINE 4 B - 1 GiB) on the fused kernel,
    4 ranks on this GPU: every byte of every rank equals the root's."""
    n, m = 4, 1 << 30
    if torch.cuda.get_device_properties(0).total_memory < 6 * m:
        pytest.skip("needs 6 GiB of device memory")
    g = torch.Generator(device="cuda:0").manual_seed(root + 11)
    bufs = [torch.zeros(m, dtype=torch.uint8, device="cuda:0") for _ in range(n)]
    bufs[root].copy_(torch.randint(0, 256, (m,), dtype=torch.uint8, device="cuda:0", generator=g))
    B.run_bcast(comms_for(n), root, bufs, m, cfg_of("chain_pipelined", chunk))
    for r in range(n):
        assert torch.equal(bufs[r], bufs[root]), r
    del bufs
    torch.cuda.empty_cache()


@pytest.mark.parametrize("claim", [1, 0])
def test_fused_chain_claimed_items_back_to_back_and_two_streams(claim):
    """The fused single-GPU kernel claims items from a per-launch counter that
    its last claimer re-zeroes: 60 back-to-back calls of changing size, item
    size and root (no host sync between them), then calls on two streams that
    may overlap (each launch owns its own counter), every byte checked."""
    n = 4
    comms = comms_for(n, {"local_claim": claim})
    assert comms[0].path(1 << 20, cfg_of("chain_pipelined", 65536)) == "local_chain_kernel"
    rng = random.Random(61 + claim)
    cap = 9 << 20
    bufs = [torch.zeros(cap, dtype=torch.uint8, device="cuda:0") for _ in range(n)]
    expect = []
    for it in range(60):
        m = rng.choice([rng.randrange(1, 5000), rng.randrange(5000, 1 << 20), rng.randrange(1 << 20, cap + 1)])
        root = rng.randrange(n)
        bufs[root][:m].fill_((it * 13 + 1) & 0xFF)
        B.bcast_all(comms, [b[:m] for b in bufs], m, "uint8", root, cfg_of("chain_pipelined", rng.choice([4096, 65536, 524288])))
        expect.append((m, (it * 13 + 1) & 0xFF))
        if it % 10 == 9:
            torch.cuda.synchronize()
            for r in range(n):
                assert int(bufs[r][:m].min()) == expect[-1][1] == int(bufs[r][:m].max()), (it, m, r)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    other = [torch.zeros(cap, dtype=torch.uint8, device="cuda:0") for _ in range(n)]
    torch.cuda.synchronize()
    for it in range(8):
        for k, (bs, st) in enumerate(((bufs, s1), (other, s2))):
            with torch.cuda.stream(st):
                bs[0].fill_(100 + 2 * it + k)
            B.bcast_all(comms, bs, cap, "uint8", 0, cfg_of("chain_pipelined", 524288), streams=[st] * n)
    torch.cuda.synchronize()
    for k, bs in enumerate((bufs, other)):
        for r in range(n):
            assert int(bs[r].min()) == 100 + 14 + k == int(bs[r].max()), (k, r)
    for c in comms:
        c.check()


@pytest.mark.parametrize("variant", ["auto", "xpull", "xpush", "ll128"])
def test_back_to_back_calls_change_payload_and_root(variant):
    """Epoch stress: buffers reused immediately, roots and payloads vary; the
    chain calls run on the variant's device path."""
    n, m = 4, 3 << 20
    options, proto = VARIANTS[variant]
    comms = comms_for(n, options)
    bufs = [torch.zeros(m, dtype=torch.uint8, device="cuda:0") for _ in range(n)]
    try:
        for it in range(40):
            root = it % n
            bufs[root].fill_(it + 1)
            algo = ["chain_pipelined", "knomial", "scatter_ring_allgather", "direct"][it % 4]
            for c in comms:
                c.set_protocol(proto if algo == "chain_pipelined" else "auto")
            B.bcast_all(comms, bufs, m, "uint8", root, cfg_of(algo, 262144 + it, 2))
            if it % 7 == 6:
                torch.cuda.synchronize()
                for r in range(n):
                    assert int(bufs[r].min()) == it + 1 == int(bufs[r].max()), (it, r)
        torch.cuda.synchronize()
        for c in comms:
            c.check()
    finally:
        for c in comms:
            c.set_protocol("auto")


@pytest.mark.parametrize("n", [2, 4, 7])
def test_ll128_direct_lines_one_gpu(n):
    """LL128 lines for the `direct` schedule (what runs across GPUs from 128
    KiB up to the LL threshold), here through L2 with the ll128=1 option:
    sizes around the threshold and the 120-byte line payload, every root,
    misaligned views against the oracle, then back-to-back calls alternating
    with 16-byte LL direct lines on the same halves."""
    comms = comms_for(n, VARIANTS["ll128"][0])
    d = cfg_of("direct")
    assert comms[0].path(128 << 10, d) == comms[0].path(2 << 20, d) == "ll128_kernel/direct"
    assert comms[0].path((128 << 10) - 1, d) == "ll_kernel/direct"
    for root in range(n):
        for m in ((128 << 10), 120 * 1200 + 1, (1 << 20) + 3, 2 << 20):
            run_case("direct", n, root, m, seed=m + root, protocol="ll128")
    run_case("direct", n, n - 1, (700 << 10) + 5, seed=3, offsets=[(5 * r) % 16 for r in range(n)], protocol="ll128")
    bufs = [torch.zeros(2 << 20, dtype=torch.uint8, device="cuda:0") for _ in range(n)]
    for it in range(30):
        m = [(1 << 20) + it, 5000 + it, (2 << 20) - it, 131072 + 120 * it][it % 4]
        root = (it * 3) % n
        for r in range(n):
            bufs[r][:m].fill_(it + 1 if r == root else 0)
        B.bcast_all(comms, [b[:m] for b in bufs], m, "uint8", root, d)
        torch.cuda.synchronize()
        for r in range(n):
            assert int(bufs[r][:m].min()) == it + 1 == int(bufs[r][:m].max()), (it, m, root, r)
    for c in comms:
        c.check()


def test_provenance_matches_schedule_sends():
    """Schedule fidelity (test_runtime.cpp:121-161): every (src, dst, chunk)
    pull happened once and moved exactly the chunk's bytes."""
    n, m = 6, 50000
    for algo, chunk, variant in (("scatter_ring_allgather", 0, "auto"), ("chain_pipelined", 7000, "auto"),
                                 ("chain_pipelined", 7000, "pull"), ("chain_pipelined", 8192, "xpull"),
                                 ("chain_pipelined", 7000, "xpull"), ("knomial", 0, "auto")):
        cfg = cfg_of(algo, chunk, 2)
        sched = B.make_schedule(cfg, n, 2, m)
        k = len(sched.chunks)
        options, protocol = VARIANTS[variant]
        comms = comms_for(n, options)
        prov = [torch.zeros(n * k, dtype=torch.int64, device="cuda:0") for _ in range(n)]
        for r in range(n):
            comms[r].set_provenance(prov[r])
            comms[r].set_protocol(protocol)  # chain: auto = the fused kernel, pull = the lane executor
        payload = O.payload(3, m)
        _, views = make_bufs(n, m, 2, payload)
        B.run_bcast(comms, 2, views, m, cfg)
        for r in range(n):
            comms[r].set_provenance(None)
            comms[r].set_protocol("auto")
        expected = {}
        for src, ops in enumerate(sched.per_rank_ops):
            for e in ops:
                if e.kind == "send":
                    expected[(src, e.peer, e.chunk)] = sched.chunks[e.chunk].length_bytes
        got = {}
        for dst in range(n):
            cnt = prov[dst].view(n, k).cpu()
            for src in range(n):
                for c in range(k):
                    if int(cnt[src, c]):
                        got[(src, dst, c)] = int(cnt[src, c])
        expected = {key: v for key, v in expected.items() if v}
        assert got == expected, (algo, variant)


def test_auto_config_uses_table_select():
    n = 4
    comms = comms_for(n)
    for m in (4, 4096, 1 << 20, 8 << 20):
        want = B.select(B.builtin_table(), n, m)
        got = comms[0].choose(m)
        assert got.algorithm == want.algorithm
        if want.algorithm == B.Algorithm.chain_pipelined:
            assert got.chunk_bytes == max(1, min(want.chunk_bytes, max(m, 1)))
        payload = O.payload(m, m)
        _, views = make_bufs(n, m, 3, payload)
        B.bcast_all(comms, views, m, "uint8", 3, None)
        torch.cuda.synchronize()
        for r in range(n):
            assert views[r].cpu().numpy().tobytes() == payload


def test_dtype_count_and_nan_payloads_are_bit_exact():
    """float32 payloads holding NaN / denormal bit patterns move untouched."""
    n, count = 4, 1 << 18
    comms = comms_for(n)
    bits = torch.randint(-(1 << 31), (1 << 31) - 1, (count,), dtype=torch.int32, device="cuda:0")
    bits[::7] = 0x7FC00001  # NaN with payload
    bits[1::11] = 0x00000001  # denormal
    bufs = [torch.zeros(count, dtype=torch.float32, device="cuda:0") for _ in range(n)]
    bufs[2].copy_(bits.view(torch.float32))
    B.bcast_all(comms, bufs, count, "float32", 2, cfg_of("chain_pipelined", 65536))
    torch.cuda.synchronize()
    for r in range(n):
        assert torch.equal(bufs[r].view(torch.int32), bits)


def test_host_buffer_run_bcast_pieces():
    """Host-buffer run_bcast pipelines 4 MiB pieces: > 2 pieces, ragged end."""
    n, m = 3, (9 << 20) + 13
    comms = B.Comm.local([0] * n, timeout_s=10)
    payload = O.payload(5, m)
    hosts = [bytearray(m) for _ in range(n)]
    hosts[2][:] = payload
    B.run_bcast_host(comms, 2, hosts, m, None)
    for r in range(n):
        assert bytes(hosts[r]) == payload


def test_host_buffer_run_bcast():
    n, m = 4, 777777
    comms = B.Comm.local([0] * n, timeout_s=10)
    payload = O.payload(4, m)
    hosts = [bytearray(m) for _ in range(n)]
    hosts[1][:] = payload
    wall = B.run_bcast_host(comms, 1, hosts, m, cfg_of("chain_pipelined", 131072))
    assert wall > 0
    for r in range(n):
        assert bytes(hosts[r]) == payload


def test_options_are_validated():
    with pytest.raises(ValueError):
        B.Comm.local([0, 0], bogus_knob=1)
    with pytest.raises(ValueError, match="shared memory"):  # 4 x 8 KiB stages x 8 warps > 227 KiB
        B.Comm.local([0, 0], stage_bytes=8192, stages=4)
    with pytest.raises(ValueError, match="nvls_slot"):
        B.Comm.local([0, 0], nvls_slot=3000)
    # LL128 direct: threshold and grid knobs; 0 turns the lines off, a threshold above the LL cap too
    d = cfg_of("direct")
    assert B.Comm.local([0, 0], ll128=1, ll128_direct_min=0)[0].path(1 << 20, d) == "ll_kernel/direct"
    assert B.Comm.local([0, 0], ll128=1, ll128_direct_min=64 << 20)[0].path(2 << 20, d) == "ll_kernel/direct"
    small = B.Comm.local([0, 0], ll128=1, ll128_direct_min=4096, ll128_direct_ctas=8)
    assert small[0].path(4096, d) == "ll128_kernel/direct"
    bufs = [torch.full((100003,), 7 if r == 1 else 0, dtype=torch.uint8, device="cuda:0") for r in range(2)]
    B.bcast_all(small, bufs, 100003, "uint8", 1, d)  # ~834 lines on 8 CTAs: every warp loops
    torch.cuda.synchronize()
    assert all(int(b.min()) == 7 == int(b.max()) for b in bufs)
    assert B.Comm.local([0, 0])[0].path(1 << 20, d) == "ll_kernel/direct"  # shared GPU without ll128=1
    comms = comms_for(2)  # ranks sharing a GPU: LL128 only with the ll128=1 option
    bufs = [torch.zeros(16, dtype=torch.uint8, device="cuda:0") for _ in comms]
    for c in comms:
        c.set_protocol("ll128")
    try:
        with pytest.raises(ValueError):
            B.bcast_all(comms, bufs, 16, "uint8", 0, cfg_of("chain_pipelined", 4))
    finally:
        for c in comms:
            c.set_protocol("auto")


def test_contract_errors():
    comms = comms_for(2)
    buf = torch.zeros(16, dtype=torch.uint8, device="cuda:0")
    with pytest.raises(ValueError):
        B.bcast_all(comms, [buf, buf], 16, "uint8", 2, cfg_of("chain"))  # root out of range
    with pytest.raises(ValueError):
        B.bcast_all(comms, [buf, buf], 16, "uint8", 0, B.AlgorithmConfig(B.Algorithm.chain_pipelined, 0, 0))
    with pytest.raises(ValueError):
        comms[0].bcast(buf, 16, "uint8", 0, cfg_of("chain"))  # ranks share a GPU: per-rank call refused
    one = B.Comm.local([0])
    with pytest.raises(ValueError):  # schedules.cpp:164-166
        B.run_bcast(one, 0, [buf], 16, cfg_of("chain_pipelined", 4))
    B.run_bcast(one, 0, [buf], 16, cfg_of("chain"))  # n = 1: untouched, no error


def test_ll_small_direct_back_to_back_reuse():
    """LL protocol (direct, <= 64 KiB): landing halves alternate by epoch and
    are reused every other call; roots and sizes change every call and every
    call is verified before the next is issued on the same buffers."""
    n = 5
    comms = comms_for(n)
    rng = random.Random(77)
    bufs = [torch.zeros(65536 + 64, dtype=torch.uint8, device="cuda:0") for _ in range(n)]
    for it in range(60):
        m = rng.choice([0, 1, 7, 8, 9, 4096, 65535, 65536, rng.randrange(1, 65537)])
        root = rng.randrange(n)
        off = rng.choice([0, 0, 3])
        views = [b[off:off + m] for b in bufs]
        payload = O.payload(it, m)
        for r in range(n):
            views[r].zero_()
        if m:
            views[root].copy_(torch.frombuffer(bytearray(payload), dtype=torch.uint8))
        B.bcast_all(comms, views, m, "uint8", root, cfg_of("direct"))
        torch.cuda.synchronize()
        for r in range(n):
            assert views[r].cpu().numpy().tobytes() == payload, (it, m, root, r)
    for c in comms:
        c.check()


@pytest.mark.parametrize("model,bucket", [("lenet", 0), ("alexnet", 0), ("alexnet", 1 << 20), ("resnet50", 4 << 20)])
def test_layerwise_parameter_broadcast(model, bucket):
    """BASELINE configs 4/5 shape: every parameter tensor broadcast from a
    non-zero root with the tuned algorithm per tensor size."""
    from paper_1707_09414_b200.params import ParamBroadcaster
    from paper_1707_09414_b200.workloads import MODELS
    n, root = 4, 3
    pb = ParamBroadcaster(MODELS[model], bucket_bytes=bucket)
    comms = comms_for(n)
    g = torch.Generator(device="cuda:0").manual_seed(len(pb))
    flats = [torch.zeros(pb.total_bytes, dtype=torch.uint8, device="cuda:0") for _ in range(n)]
    flats[root].copy_(torch.randint(0, 256, (pb.total_bytes,), dtype=torch.uint8, device="cuda:0", generator=g))
    torch.cuda.synchronize()
    pb.bcast_all(comms, flats, root)
    torch.cuda.synchronize()
    for r in range(n):
        for off, size in zip(pb.offsets, pb.sizes):
            assert torch.equal(flats[r][off:off + size], flats[root][off:off + size]), (model, r, off)


def test_protocol_caps_and_lane_plan():
    """bcl_comm_protocol_caps / bcl_comm_plan on a single-GPU group: no LL128
    (ranks share the GPU), LL caps as configured; the lane plan tiles the
    lanes (Q divides L) and covers each chunk with Q slices."""
    comms = comms_for(4)
    caps = comms[0].protocol_caps()
    assert caps == {"ll_direct": 2 << 20, "ll_chain": 8 << 20, "ll128": 0}
    assert comms_for(4, VARIANTS["ll128"][0])[0].protocol_caps()["ll128"] == 32 << 20
    # the device path each variant runs (bcl_comm_path)
    chain = cfg_of("chain_pipelined", 65536)
    want = {"auto": "local_chain_kernel", "pull": "bcast_kernel/pull", "ll": "ll_kernel/chain",
            "push": "bcast_kernel/push", "xpull": "bcast_kernel/pull/tma", "xstrict": "bcast_kernel/pull/tma",
            "xpush": "bcast_kernel/push/tma", "ll128": "ll128_kernel"}
    for variant, (options, proto) in VARIANTS.items():
        c = comms_for(4, options)[0]
        c.set_protocol(proto)
        try:
            assert c.path(1 << 20, chain) == want[variant], variant
        finally:
            c.set_protocol("auto")
    assert comms[0].path(4096, cfg_of("direct")) == "ll_kernel/direct"
    assert comms[0].path(4096, cfg_of("knomial", radix=2)) == "bcast_kernel/events"
    lanes = comms[0].info()["lanes"]
    for m, chunk in ((64 << 20, 512 << 10), (1 << 20, 65536), (12345, 1000)):
        p = comms[0].plan(cfg_of("chain_pipelined", chunk), 0, m)
        assert lanes % p["slices"] == 0
        assert p["n_chunks"] == -(-m // chunk)
        assert p["slices"] * p["slice_bytes"] >= min(chunk, m)
        assert 1 <= p["ctas"] * 8 <= lanes


def _grouped_round(comms, bufs, sizes, root, algo, chunk=65536, offs=None):
    """Issue one broadcast per size inside one bcl_group_start/end; returns
    the expected payload per message."""
    n = len(comms)
    expect = []
    at = 0
    views = []
    for k, m in enumerate(sizes):
        off = at + (offs[k] if offs else 0)
        views.append([b[off:off + m] for b in bufs])
        at = off + m + 16
    for k, m in enumerate(sizes):
        src = torch.randint(0, 256, (m,), dtype=torch.uint8, device=bufs[root].device)
        for r in range(n):
            (views[k][r].copy_(src) if r == root else views[k][r].fill_(0x3C))
        expect.append(src)
    torch.cuda.synchronize()
    with B.group():
        for k, m in enumerate(sizes):
            B.bcast_all(comms, views[k], m, "uint8", root, cfg_of(algo, chunk))
    torch.cuda.synchronize()
    for k in range(len(sizes)):
        for r in range(n):
            assert torch.equal(views[k][r], expect[k]), (algo, sizes[k], r)


def test_group_fuses_line_protocol_calls():
    """bcl_group_start/end: consecutive LL direct calls (and LL chain calls
    under protocol ll) share launches, with
    odd sizes, misaligned views and an empty message, bit-exact (8 messages
    per launch when ranks share a GPU: 40 in 5 launches); calls that
    cannot fuse (the fused single-GPU chain) run as usual, in order."""
    n = 4
    comms = comms_for(n)
    bufs = [torch.zeros(8 << 20, dtype=torch.uint8, device="cuda:0") for _ in range(n)]
    rng = random.Random(71)
    sizes = [rng.choice([1, 7, 8, 9, 255, 4096, rng.randrange(1, 100000)]) for _ in range(39)] + [0]
    before = comms[0].launches
    _grouped_round(comms, bufs, sizes, 2, "direct", offs=[rng.randrange(0, 8) for _ in sizes])
    assert comms[0].launches - before == 5  # 40 messages, 8 per launch on a shared GPU
    # mixed: direct (fusable) and chain (fused single-GPU kernel, not fusable)
    before = comms[0].launches
    sizes = [1000, 2000, 3000]
    at = 0
    views = []
    for m in sizes + [1 << 20] + sizes:
        views.append([b[at:at + m] for b in bufs])
        at += m + 64
    for r in range(n):
        for v in views:
            (v[r].fill_(0x11) if r == 1 else v[r].zero_())
    torch.cuda.synchronize()
    with B.group():
        for k, v in enumerate(views):
            algo = "chain_pipelined" if k == 3 else "direct"
            B.bcast_all(comms, v, v[0].numel(), "uint8", 1, cfg_of(algo, 65536))
    torch.cuda.synchronize()
    assert comms[0].launches - before == 3
    for v in views:
        for r in range(n):
            assert int(v[r].min()) == 0x11 == int(v[r].max())
    for c in comms:
        c.set_protocol("ll")
    try:
        before = comms[0].launches
        _grouped_round(comms, bufs, [5, 100, 65536, 3 << 20, 17], 0, "chain_pipelined")
        assert comms[0].launches - before == 1
    finally:
        for c in comms:
            c.set_protocol("auto")


@pytest.mark.parametrize("n", [2, 4])
def test_group_fuses_ll128_direct_lines(n):
    """A group whose `direct` run holds a message >= ll128_direct_min travels
    on LL128 direct lines, every member a segment (small and large, odd
    sizes, misaligned, an empty one): one launch per run, bit-exact; a run of
    small messages only stays on 16-byte LL lines."""
    comms = comms_for(n, VARIANTS["ll128"][0])
    bufs = [torch.zeros(4 << 20, dtype=torch.uint8, device="cuda:0") for _ in range(n)]
    rng = random.Random(5 + n)
    sizes = [1, 119, 120, 121, 300000, 0, 4096 + 7, 131072]  # (ranks sharing a GPU: <= 8 messages per launch)
    before = comms[0].launches
    _grouped_round(comms, bufs, sizes, n - 1, "direct", offs=[rng.randrange(0, 8) for _ in sizes])
    assert comms[0].launches - before == 1
    before = comms[0].launches
    _grouped_round(comms, bufs, [(700 << 10) + 3, 5, (900 << 10) + 1], 0, "direct", offs=[3, 0, 1])
    assert comms[0].launches - before == 1
    # beyond the LL128 direct area (~2 MiB of lines): the run splits
    before = comms[0].launches
    _grouped_round(comms, bufs, [(1 << 20) + 9, (1 << 20) + 11, 1000], 1 % n, "direct")
    assert comms[0].launches - before == 2
    for c in comms:
        c.check()


def test_group_rules():
    comms = comms_for(2)
    buf = [torch.zeros(64, dtype=torch.uint8, device="cuda:0") for _ in comms]
    with pytest.raises(ValueError):
        B._lib._check(B.lib().bcl_group_end())  # end without start
    with pytest.raises(ValueError):
        with B.group():
            B.run_bcast(comms, 0, buf, 64, cfg_of("direct"))
    with B.group():
        with B.group():  # nested: fused at the outermost end
            B.bcast_all(comms, buf, 64, "uint8", 0, cfg_of("direct"))
        B.bcast_all(comms, buf, 64, "uint8", 0, cfg_of("direct"))
    torch.cuda.synchronize()


@pytest.mark.parametrize("model", ["resnet50", "lenet"])
def test_layerwise_parameter_broadcast_fused(model):
    """Configs 4/5 with the per-tensor broadcasts grouped: still one message
    per tensor, far fewer launches, every tensor bit-exact."""
    from paper_1707_09414_b200.params import ParamBroadcaster
    from paper_1707_09414_b200.workloads import MODELS
    n, root = 4, 1
    pb = ParamBroadcaster(MODELS[model], fused=True)
    comms = comms_for(n)
    g = torch.Generator(device="cuda:0").manual_seed(7)
    flats = [torch.zeros(pb.total_bytes, dtype=torch.uint8, device="cuda:0") for _ in range(n)]
    flats[root].copy_(torch.randint(0, 256, (pb.total_bytes,), dtype=torch.uint8, device="cuda:0", generator=g))
    torch.cuda.synchronize()
    before = comms[0].launches
    pb.bcast_all(comms, flats, root)
    torch.cuda.synchronize()
    assert comms[0].launches - before < len(pb)
    for r in range(n):
        for off, size in zip(pb.offsets, pb.sizes):
            assert torch.equal(flats[r][off:off + size], flats[root][off:off + size]), (model, r, off)


@pytest.mark.parametrize("variant", ["auto", "pull", "ll", "xpull", "xpush", "ll128"])
def test_graph_capture_replays_fresh_epochs(variant):
    """Epochs and the line protocols' reuse bookkeeping live on the device
    (CallState), so a CUDA graph of broadcasts replays correctly: a captured
    sequence (a chain call on the variant's path, a small direct call, a
    device barrier, a grouped pair) replayed 6 times with a fresh payload
    each time, interleaved with eager calls, every byte checked."""
    n, m = 4, (1 << 20) + 3
    options, proto = VARIANTS[variant]
    comms = comms_for(n, options)
    for c in comms:
        c.set_protocol(proto)
    try:
        bufs = [torch.zeros(m, dtype=torch.uint8, device="cuda:0") for _ in range(n)]
        small = [torch.zeros(777, dtype=torch.uint8, device="cuda:0") for _ in range(n)]
        pair = [[torch.zeros(k, dtype=torch.uint8, device="cuda:0") for _ in range(n)] for k in (100, 5000)]
        s = torch.cuda.Stream()
        chain = cfg_of("chain_pipelined", 65536)

        def body():
            B.bcast_all(comms, bufs, m, "uint8", 1, chain, streams=[s] * n)
            B.bcast_all(comms, small, 777, "uint8", 2, cfg_of("direct"), streams=[s] * n)
            B.barrier_all(comms, streams=[s] * n)
            with B.group():
                for p in pair:
                    B.bcast_all(comms, p, p[0].numel(), "uint8", 3, cfg_of("direct"), streams=[s] * n)

        with torch.cuda.stream(s):
            body()  # warm-up outside capture (lazy allocations happen here)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            body()
        torch.cuda.synchronize()
        for rep in range(6):
            vals = [(rep * 4 + k) % 251 + 1 for k in range(4)]
            for r in range(n):
                bufs[r].fill_(vals[0] if r == 1 else 0)
                small[r].fill_(vals[1] if r == 2 else 0)
                for k, p in enumerate(pair):
                    p[r].fill_(vals[2 + k] if r == 3 else 0)
            torch.cuda.synchronize()
            with torch.cuda.stream(s):  # (calls on one communicator must be ordered: one stream)
                g.replay()
                if rep % 2:  # eager calls between replays keep the device state moving
                    B.bcast_all(comms, small, 777, "uint8", 2, cfg_of("direct"), streams=[s] * n)
            torch.cuda.synchronize()
            for r in range(n):
                assert int(bufs[r].min()) == vals[0] == int(bufs[r].max()), (variant, rep, r)
                assert int(small[r].min()) == vals[1] == int(small[r].max()), (variant, rep, r)
                for k, p in enumerate(pair):
                    assert int(p[r].min()) == vals[2 + k] == int(p[r].max()), (variant, rep, k, r)
        for c in comms:
            c.check()
    finally:
        for c in comms:
            c.set_protocol("auto")
