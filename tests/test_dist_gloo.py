"""N>1 host logic on CPU (world_size 2, gloo): the IPC-blob rendezvous used by
Comm.connect_torch and the max-over-ranks latency reduction used by bench.py."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1707_09414_b200.comm import exchange_blobs
        blobs = exchange_blobs(bytes([rank]) * (10 + rank * 0) + b"blob")
        t = torch.tensor([1.0 + rank, 5.0 - rank], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        q.put((rank, blobs, t.tolist()))
    finally:
        dist.destroy_process_group()


def test_blob_exchange_and_max_reduction_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, blobs, t in out:
        assert blobs == [bytes([0]) * 10 + b"blob", bytes([1]) * 10 + b"blob"]
        assert t == [2.0, 5.0]
