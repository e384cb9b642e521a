"""Communicator and data plane (the TransportFabric / run_bcast boundary,
proj/include/bcastlab/runtime.hpp:20-143) over libbcl.so.

Buffers are device pointers (int) or CUDA tensors; streams are raw
cudaStream_t handles (int) or torch.cuda.Stream objects. torch is only used
here for plumbing (device memory, streams, the rendezvous of the IPC blobs).
"""
import ctypes as C
from typing import List, Optional, Sequence

from ._lib import AlgorithmConfig, DTYPES, _Config, _check, lib


def _ptr(x) -> int:
    if x is None:
        return 0
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return int(x.data_ptr())
    raise TypeError(f"expected a device pointer or tensor, got {type(x)!r}")


def _stream(s) -> Optional[int]:
    if s is None:
        return None
    if isinstance(s, int):
        return s
    if hasattr(s, "cuda_stream"):
        return int(s.cuda_stream)
    raise TypeError(f"expected a cudaStream_t or torch.cuda.Stream, got {type(s)!r}")


def _dtype(d) -> int:
    if isinstance(d, int):
        return d
    return DTYPES[str(d).replace("torch.", "")]


def _options(timeout_s, options) -> bytes:
    items = dict(options)
    if timeout_s and timeout_s > 0:
        items.setdefault("timeout_s", timeout_s)
    return ",".join(f"{k}={int(v) if isinstance(v, bool) else v}" for k, v in items.items()).encode()


def _cfg(config: Optional[AlgorithmConfig]):
    return C.byref(config._c()) if config is not None else None


class DevicePtr:
    """Raw device memory as a __cuda_array_interface__ object, so
    torch.as_tensor(DevicePtr(p, n), device='cuda') views it without a copy."""

    def __init__(self, ptr: int, nbytes: int):
        self.ptr, self.nbytes = ptr, nbytes

    @property
    def __cuda_array_interface__(self):
        return {"shape": (self.nbytes,), "typestr": "|u1", "data": (self.ptr, False), "version": 3}


class Comm:
    """One rank's handle (bcl_comm_t)."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle

    # ------------------------------------------------------------ creation
    @staticmethod
    def local(devices: Sequence[int], timeout_s: float = 0.0, **options) -> List["Comm"]:
        """One process drives len(devices) ranks (rank r on devices[r]).
        options: communicator options of bcl_comm_init_all_opts (include/bcl.h),
        e.g. stage_bytes=8192, sys_scope=1, ll128=1."""
        n = len(devices)
        out = (C.c_void_p * n)()
        devs = (C.c_int * n)(*devices)
        if options:
            _check(lib().bcl_comm_init_all_opts(n, devs, _options(timeout_s, options), out))
        else:
            _check(lib().bcl_comm_init_all(n, devs, timeout_s, out))
        return [Comm(C.c_void_p(out[i])) for i in range(n)]

    @staticmethod
    def rank(n: int, rank: int, device: int, heap_bytes: int = 0, timeout_s: float = 0.0, **options) -> "Comm":
        """One process per GPU; call export()/connect() (or use connect_torch)."""
        h = C.c_void_p()
        if options:
            _check(lib().bcl_comm_init_rank_opts(n, rank, device, heap_bytes, _options(timeout_s, options),
                                                 C.byref(h)))
        else:
            _check(lib().bcl_comm_init_rank(n, rank, device, heap_bytes, timeout_s, C.byref(h)))
        return Comm(h)

    @staticmethod
    def connect_torch(n: int, rank: int, device: int, heap_bytes: int = 0, timeout_s: float = 0.0,
                      group=None, **options) -> "Comm":
        """init_rank + an all_gather of the IPC blobs over torch.distributed."""
        c = Comm.rank(n, rank, device, heap_bytes, timeout_s, **options)
        c.connect(exchange_blobs(c.export(), group))
        return c

    def export(self) -> bytes:
        ln = C.c_size_t()
        _check(lib().bcl_comm_export(self._h, None, 0, C.byref(ln)))
        buf = C.create_string_buffer(ln.value)
        _check(lib().bcl_comm_export(self._h, buf, ln.value, C.byref(ln)))
        return buf.raw[:ln.value]

    def connect(self, blobs: Sequence[bytes]) -> None:
        size = len(blobs[0])
        if any(len(b) != size for b in blobs):
            raise ValueError("info blobs differ in size")
        joined = b"".join(blobs)
        _check(lib().bcl_comm_connect(self._h, C.c_char_p(joined), size))

    def register(self, buf, nbytes: Optional[int] = None, group=None) -> None:
        """Collective (per-process ranks): register the device allocation
        holding `buf` so broadcasts on buffers inside it are zero-copy; the
        blobs are exchanged over torch.distributed. No-op for one-process groups."""
        nbytes = nbytes if nbytes is not None else (buf.numel() * buf.element_size() if hasattr(buf, "numel") else 0)
        ln = C.c_size_t()
        _check(lib().bcl_comm_register_export(self._h, C.c_void_p(_ptr(buf)), nbytes, None, 0, C.byref(ln)))
        if ln.value == 0:
            return
        blob = C.create_string_buffer(ln.value)
        _check(lib().bcl_comm_register_export(self._h, C.c_void_p(_ptr(buf)), nbytes, blob, ln.value, C.byref(ln)))
        blobs = exchange_blobs(blob.raw[:ln.value], group)
        joined = b"".join(blobs)
        _check(lib().bcl_comm_register_connect(self._h, C.c_char_p(joined), ln.value))

    def close(self) -> None:
        if self._h is not None and self._h.value:
            lib().bcl_comm_destroy(self._h)
            self._h = None

    # -------------------------------------------------------------- queries
    def info(self):
        n, r, d, l = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        _check(lib().bcl_comm_info(self._h, C.byref(n), C.byref(r), C.byref(d), C.byref(l)))
        return {"n": n.value, "rank": r.value, "device": d.value, "lanes": l.value}

    def protocol_caps(self):
        """Largest message (bytes, 0 = unavailable) per line protocol."""
        d, c, l128 = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(lib().bcl_comm_protocol_caps(self._h, C.byref(d), C.byref(c), C.byref(l128)))
        return {"ll_direct": d.value, "ll_chain": c.value, "ll128": l128.value}

    @property
    def n_ranks(self) -> int:
        return self.info()["n"]

    @property
    def rank_id(self) -> int:
        return self.info()["rank"]

    def set_table(self, table) -> None:
        _check(lib().bcl_comm_set_table(self._h, table._h))

    def plan(self, config: AlgorithmConfig, root: int, nbytes: int) -> dict:
        """Device lane plan of a call: slices per chunk, slice bytes, chunks, CTAs."""
        q, sb, nc, ctas = C.c_int(), C.c_uint64(), C.c_uint32(), C.c_int()
        _check(lib().bcl_comm_plan(self._h, C.byref(config._c()), root, nbytes, C.byref(q), C.byref(sb),
                                   C.byref(nc), C.byref(ctas)))
        return {"slices": q.value, "slice_bytes": sb.value, "n_chunks": nc.value, "ctas": ctas.value}

    def nvls(self):
        """(available, reason): the communicator's NVLS multicast team (every rank agrees)."""
        ok, ln = C.c_int(), C.c_size_t()
        _check(lib().bcl_comm_nvls(self._h, C.byref(ok), None, 0, C.byref(ln)))
        buf = C.create_string_buffer(ln.value)
        _check(lib().bcl_comm_nvls(self._h, C.byref(ok), buf, ln.value, C.byref(ln)))
        return bool(ok.value), buf.value.decode()

    PROTOCOLS = {"auto": 0, "pull": 1, "push": 2, "ll": 3, "ll128": 4, "nvls": 5}

    def set_protocol(self, protocol) -> None:
        """Transport: "auto" (LL128/LL up to their caps, then the table rule), "pull", "push", "ll", "ll128"
        or "nvls" (NVLS multicast, any schedule)."""
        code = self.PROTOCOLS[protocol] if isinstance(protocol, str) else int(protocol)
        _check(lib().bcl_comm_set_protocol(self._h, code))

    def path(self, nbytes: int, config: Optional[AlgorithmConfig] = None, root: int = 0) -> str:
        """The device path (kernel/protocol) a call of this shape runs."""
        ln = C.c_size_t()
        cc = _cfg(config)
        _check(lib().bcl_comm_path(self._h, cc, root, nbytes, None, 0, C.byref(ln)))
        buf = C.create_string_buffer(ln.value)
        _check(lib().bcl_comm_path(self._h, cc, root, nbytes, buf, ln.value, C.byref(ln)))
        return buf.value.decode()

    def choose(self, message_bytes: int) -> AlgorithmConfig:
        out = _Config()
        _check(lib().bcl_comm_choose(self._h, message_bytes, C.byref(out)))
        return AlgorithmConfig._from(out)

    def alloc(self, nbytes: int) -> int:
        p = C.c_void_p()
        _check(lib().bcl_mem_alloc(self._h, nbytes, C.byref(p)))
        return int(p.value or 0)

    def reset_heap(self) -> None:
        _check(lib().bcl_mem_reset(self._h))

    @property
    def launches(self) -> int:
        v = C.c_uint64()
        _check(lib().bcl_comm_launches(self._h, C.byref(v)))
        return v.value

    # ---------------------------------------------------------- data plane
    def bcast(self, buf, count: int, dtype="uint8", root: int = 0,
              config: Optional[AlgorithmConfig] = None, stream=None) -> None:
        """bcast(buf, count, dtype, root, comm): enqueued on `stream`. (The
        per-call path is kept lean: a training step issues one per tensor.)"""
        status = lib().bcl_bcast(_ptr(buf), count, _dtype(dtype), root, self._h,
                                 None if config is None else C.byref(config._c()), _stream(stream))
        if status:
            _check(status)

    def bcast_host(self, host_buf, count: int, dtype="uint8", root: int = 0,
                   config: Optional[AlgorithmConfig] = None, stream=None) -> None:
        _check(lib().bcl_bcast_host(C.c_void_p(_ptr(host_buf)), count, _dtype(dtype), root, self._h,
                                    _cfg(config), C.c_void_p(_stream(stream))))

    def barrier(self, stream=None) -> None:
        _check(lib().bcl_barrier(self._h, C.c_void_p(_stream(stream))))

    def check(self, stream=None) -> None:
        _check(lib().bcl_comm_check(self._h, C.c_void_p(_stream(stream))))

    def set_trace(self, records, per_lane: int = 0) -> None:
        """records: int64 device tensor of lanes * per_lane * 4 stamps (or None)."""
        _check(lib().bcl_comm_set_trace(self._h, C.c_void_p(_ptr(records)), per_lane if records is not None else 0))

    def set_provenance(self, counters) -> None:
        _check(lib().bcl_comm_set_provenance(self._h, C.c_void_p(_ptr(counters))))


class group:
    """``with group(): ...`` -- bcl_group_start/end (NCCL-style fusion): the
    broadcasts issued inside are deferred and, at the end, consecutive ones on
    the same line protocol, root and stream are fused into one launch."""

    def __enter__(self):
        _check(lib().bcl_group_start())
        return self

    def __exit__(self, exc_type, exc, tb):
        status = lib().bcl_group_end()
        if exc_type is None:
            _check(status)
        return False


def exchange_blobs(blob: bytes, group=None) -> List[bytes]:
    """All-gather one opaque blob per rank (ordered by rank) over an
    initialised torch.distributed group (any backend; plumbing only)."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, bytes(blob), group=group)
    if any(not isinstance(b, (bytes, bytearray)) for b in out):
        raise ValueError("a rank contributed no blob")
    return [bytes(b) for b in out]


def _handles(comms: Sequence[Comm]):
    return (C.c_void_p * len(comms))(*[c._h.value for c in comms])


def bcast_all(comms: Sequence[Comm], bufs, count: int, dtype="uint8", root: int = 0,
              config: Optional[AlgorithmConfig] = None, streams=None) -> None:
    n = len(comms)
    b = (C.c_void_p * n)(*[_ptr(x) for x in bufs])
    s = (C.c_void_p * n)(*[_stream(x) for x in streams]) if streams is not None else None
    _check(lib().bcl_bcast_all(b, count, _dtype(dtype), root, _handles(comms), n, _cfg(config), s))


def barrier_all(comms: Sequence[Comm], streams=None) -> None:
    n = len(comms)
    s = (C.c_void_p * n)(*[_stream(x) for x in streams]) if streams is not None else None
    _check(lib().bcl_barrier_all(_handles(comms), n, s))


def run_bcast(comms: Sequence[Comm], root: int, bufs, nbytes: int,
              config: Optional[AlgorithmConfig] = None) -> float:
    """run_bcast (runtime.cpp:66-103) over device buffers; returns wall s."""
    n = len(comms)
    b = (C.c_void_p * n)(*[_ptr(x) for x in bufs])
    w = C.c_double()
    _check(lib().bcl_run_bcast(n, root, b, nbytes, _cfg(config), _handles(comms), C.byref(w)))
    return w.value


def run_bcast_host(comms: Sequence[Comm], root: int, host_bufs, nbytes: int,
                   config: Optional[AlgorithmConfig] = None) -> float:
    """run_bcast over host buffers (ints, pinned tensors or bytearrays)."""
    n = len(comms)
    keep = []
    ptrs = []
    for x in host_bufs:
        if isinstance(x, (bytearray, memoryview)):
            arr = (C.c_uint8 * max(len(x), 1)).from_buffer(x)
            keep.append(arr)
            ptrs.append(C.addressof(arr))
        else:
            ptrs.append(_ptr(x))
    b = (C.c_void_p * n)(*ptrs)
    w = C.c_double()
    _check(lib().bcl_run_bcast_host(n, root, b, nbytes, _cfg(config), _handles(comms), C.byref(w)))
    return w.value
