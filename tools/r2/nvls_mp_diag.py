"""Per-process NVLS setup diagnosis: spawn W ranks (one per GPU), create the
communicator with the given options, print each rank's NVLS verdict before and
after connect, then one NVLS broadcast.

    python tools/r2/nvls_mp_diag.py [world] [options]
"""
import os
import socket
import sys

import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def worker(rank, world, port, opts):
    import torch.distributed as dist
    import paper_1707_09414_b200 as B
    from paper_1707_09414_b200.comm import exchange_blobs
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(rank)
    kw = dict(kv.split("=") for kv in opts.split(",") if kv)
    try:
        c = B.Comm.rank(world, rank, rank, 0, 10.0, **kw)
        print(f"rank {rank}: before connect nvls={c.nvls()}", flush=True)
        c.connect(exchange_blobs(c.export()))
        print(f"rank {rank}: after connect nvls={c.nvls()}", flush=True)
        if c.nvls()[0]:
            c.set_protocol("nvls")
            buf = torch.full((1 << 20,), rank, dtype=torch.uint8, device=f"cuda:{rank}")
            dist.barrier()
            c.bcast(buf, 1 << 20, "uint8", 0, B.AlgorithmConfig.of("direct"))
            c.check()
            print(f"rank {rank}: nvls bcast ok={bool((buf == 0).all())}", flush=True)
        c.close()
    except Exception as e:  # noqa: BLE001
        print(f"rank {rank}: FAILED {e!r}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    world = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    opts = sys.argv[2] if len(sys.argv) > 2 else ""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.start_processes(worker, args=(world, port, opts), nprocs=world, start_method="spawn")
