"""ctypes binding of the CPU oracle (oracle/liboracle.so) for the tests.

TEST INFRASTRUCTURE: the oracle is the checker, never the thing measured.
"""
import ctypes as C
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB_PATH = os.path.join(ROOT, "oracle", "liboracle.so")

ALGOS = ["direct", "chain", "knomial", "scatter_ring_allgather",
         "chain_pipelined", "knomial_staged"]


class Chunk(C.Structure):
    _fields_ = [("chunk_id", C.c_uint32), ("offset", C.c_uint64), ("length", C.c_uint64)]


class Event(C.Structure):
    _fields_ = [("kind", C.c_int32), ("peer", C.c_int32), ("chunk", C.c_uint32), ("group", C.c_uint32)]


class Schedule(C.Structure):
    _fields_ = [("n", C.c_int), ("root", C.c_int), ("message_bytes", C.c_uint64),
                ("prologue", C.c_int), ("n_chunks", C.c_uint32),
                ("chunks", C.POINTER(Chunk)), ("ev_off", C.POINTER(C.c_uint64)),
                ("events", C.POINTER(Event))]


class Config(C.Structure):
    _fields_ = [("algorithm", C.c_int32), ("radix_k", C.c_int32), ("chunk_bytes", C.c_uint64)]


class Entry(C.Structure):
    _fields_ = [("n", C.c_int32), ("msg_min", C.c_uint64), ("msg_max", C.c_uint64),
                ("config", Config), ("cost", C.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), os.path.join(ROOT, "oracle", "liboracle.so")],
                           check=True, capture_output=True)
        l = C.CDLL(LIB_PATH)
        l.orc_make_chunks.restype = C.c_int64
        l.orc_make_chunks.argtypes = [C.c_uint64, C.c_uint64, C.POINTER(Chunk), C.c_uint64]
        l.orc_make_schedule.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_uint64, C.POINTER(Schedule)]
        l.orc_free_schedule.argtypes = [C.POINTER(Schedule)]
        l.orc_bcast.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_uint64, C.POINTER(C.c_void_p)]
        l.orc_payload.argtypes = [C.c_uint64, C.c_uint64, C.c_void_p]
        l.orc_fnv1a.restype = C.c_uint64
        l.orc_fnv1a.argtypes = [C.c_void_p, C.c_uint64]
        l.orc_cost.restype = C.c_double
        l.orc_cost.argtypes = [C.POINTER(Config), C.c_int, C.c_uint64, C.c_double, C.c_double, C.c_double]
        l.orc_tune.restype = C.c_int64
        l.orc_tune.argtypes = [C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_uint64), C.c_int,
                               C.POINTER(Config), C.c_int, C.POINTER(C.c_uint64), C.c_int,
                               C.c_double, C.c_double, C.c_double, C.POINTER(Entry)]
        l.orc_select.argtypes = [C.POINTER(Entry), C.c_int64, C.c_int, C.c_uint64, C.POINTER(Config)]
        l.orc_save_table.restype = C.c_int64
        l.orc_save_table.argtypes = [C.POINTER(Entry), C.c_int64, C.c_int, C.c_char_p, C.c_int64]
        l.orc_load_table.restype = C.c_int64
        l.orc_load_table.argtypes = [C.c_char_p, C.POINTER(Entry), C.c_int64, C.POINTER(C.c_int)]
        l.orc_format_double.argtypes = [C.c_double, C.c_char_p, C.c_int]
        _lib = l
    return _lib


def make_chunks(m, c):
    k = lib().orc_make_chunks(m, c, None, 0)
    if k < 0:
        raise ValueError("chunk_bytes must be >= 1")
    arr = (Chunk * k)()
    lib().orc_make_chunks(m, c, arr, k)
    return [(x.chunk_id, x.offset, x.length) for x in arr]


def schedule(algo, n, root, m, chunk=0, radix=0):
    s = Schedule()
    a = ALGOS.index(algo) if isinstance(algo, str) else algo
    if lib().orc_make_schedule(a, radix, chunk, n, root, m, C.byref(s)) != 0:
        raise ValueError("invalid schedule arguments")
    chunks = [[s.chunks[i].chunk_id, s.chunks[i].offset, s.chunks[i].length] for i in range(s.n_chunks)]
    events = []
    for r in range(s.n):
        for i in range(s.ev_off[r], s.ev_off[r + 1]):
            e = s.events[i]
            events.append([r, e.kind, e.peer, e.chunk, e.group])
    out = {"prologue": s.prologue, "chunks": chunks, "events": events}
    lib().orc_free_schedule(C.byref(s))
    return out


def payload(seed, size):
    buf = (C.c_uint8 * max(size, 1))()
    lib().orc_payload(seed, size, buf)
    return bytes(buf)[:size]


def fnv(data):
    b = (C.c_uint8 * max(len(data), 1)).from_buffer_copy(data if data else b"\0")
    return lib().orc_fnv1a(b, len(data))


def bcast(algo, n, root, bufs, chunk=0, radix=0):
    """Runs the oracle broadcast in place over n bytearrays."""
    m = len(bufs[0])
    arrs = [(C.c_uint8 * max(m, 1)).from_buffer(b) if m else (C.c_uint8 * 1)() for b in bufs]
    ptrs = (C.c_void_p * n)(*[C.addressof(a) for a in arrs])
    a = ALGOS.index(algo) if isinstance(algo, str) else algo
    rc = lib().orc_bcast(a, radix, chunk, n, root, m, ptrs)
    if rc != 0:
        raise RuntimeError(f"oracle bcast failed rc={rc}")


def cost(algo, n, m, chunk=0, radix=0, ts=1e-6, bw=1e9, st=1e10):
    cfg = Config(ALGOS.index(algo), radix, chunk)
    return lib().orc_cost(C.byref(cfg), n, m, ts, bw, st)


def tune(n_list, sizes, cands, chunks, ts=1e-6, bw=1e9, st=1e10):
    nl = (C.c_int * len(n_list))(*n_list)
    sz = (C.c_uint64 * len(sizes))(*sizes)
    cf = (Config * len(cands))(*[Config(ALGOS.index(a), r, 0) for a, r in cands])
    ch = (C.c_uint64 * max(len(chunks), 1))(*chunks)
    out = (Entry * (len(n_list) * len(sizes)))()
    k = lib().orc_tune(nl, len(n_list), sz, len(sizes), cf, len(cands), ch, len(chunks), ts, bw, st, out)
    if k < 0:
        raise ValueError("invalid tune arguments")
    return [out[i] for i in range(k)]


def save_table(entries, oracle=0):
    arr = (Entry * max(len(entries), 1))(*entries)
    need = lib().orc_save_table(arr, len(entries), oracle, None, 0)
    buf = C.create_string_buffer(need + 1)
    lib().orc_save_table(arr, len(entries), oracle, buf, need + 1)
    return buf.value.decode()


def load_table(text):
    cap = 4096
    out = (Entry * cap)()
    orc = C.c_int(0)
    k = lib().orc_load_table(text.encode(), out, cap, C.byref(orc))
    if k < 0:
        return None, (0 if k == -1000000 else -k)
    return [out[i] for i in range(k)], orc.value


def select(entries, n, m):
    arr = (Entry * max(len(entries), 1))(*entries)
    cfg = Config()
    rc = lib().orc_select(arr, len(entries), n, m, C.byref(cfg))
    if rc != 0:
        return None
    return (ALGOS[cfg.algorithm], cfg.radix_k, cfg.chunk_bytes)
