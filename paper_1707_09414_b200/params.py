"""Layer-wise model-parameter broadcast: the paper's caller.

CNTK broadcasts every parameter tensor from the root before an iteration;
each tensor is one MPI_Bcast whose algorithm and chunk the tuning framework
picks from its size. `ParamBroadcaster` does the same over one flat device
buffer (each tensor 256-byte aligned): one `bcast` per tensor, or per bucket
of consecutive tensors when `bucket_bytes` > 0 (small layers coalesced into
one message, a common DL-framework optimisation). Configs 4/5 of
BASELINE.json use it with the sizes in `workloads.MODELS`.
"""
from typing import List, Optional, Sequence, Tuple

from contextlib import nullcontext

from .comm import Comm, _ptr, bcast_all, group


def layout(sizes: Sequence[int], align: int = 256) -> Tuple[List[int], int]:
    """Offsets of each tensor in a flat buffer and the buffer's total size."""
    offs, at = [], 0
    for s in sizes:
        offs.append(at)
        at += (s + align - 1) // align * align
    return offs, at


def messages(sizes: Sequence[int], bucket_bytes: int = 0, align: int = 256) -> List[Tuple[int, int]]:
    """(offset, bytes) of every broadcast: one per tensor, or buckets of
    consecutive tensors of at least `bucket_bytes` (contiguous in the flat
    buffer, alignment padding included)."""
    offs, total = layout(sizes, align)
    if bucket_bytes <= 0:
        return [(o, s) for o, s in zip(offs, sizes)]
    out, start, end = [], None, 0
    for o, s in zip(offs, sizes):
        if start is None:
            start = o
        end = o + s
        if end - start >= bucket_bytes:
            out.append((start, end - start))
            start = None
    if start is not None:
        out.append((start, end - start))
    return out


class ParamBroadcaster:
    """Broadcast a model's parameters (flat buffer) from `root`. With
    `fused`, the per-tensor broadcasts are issued inside one
    bcl_group_start/end: still one message per tensor (tuned per size), but
    runs of small ones share a launch."""

    def __init__(self, sizes: Sequence[int], bucket_bytes: int = 0, fused: bool = False):
        self.fused = fused
        self.sizes = list(sizes)
        self.msgs = messages(self.sizes, bucket_bytes)
        self.offsets, self.total_bytes = layout(self.sizes)

    def __len__(self):
        return len(self.msgs)

    def bcast(self, comm: Comm, flat, root: int, stream=None, config=None) -> None:
        """Per-rank call (one process per GPU): every rank passes its own flat buffer."""
        base = _ptr(flat)
        with group() if self.fused else nullcontext():
            for off, n in self.msgs:
                comm.bcast(base + off, n, "uint8", root, config, stream)

    def bcast_all(self, comms: Sequence[Comm], flats: Sequence, root: int, streams: Optional[Sequence] = None,
                  config=None) -> None:
        """All ranks of a one-process group."""
        bases = [_ptr(f) for f in flats]
        with group() if self.fused else nullcontext():
            for off, n in self.msgs:
                bcast_all(comms, [b + off for b in bases], n, "uint8", root, config, streams)
