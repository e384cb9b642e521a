"""ctypes binding of libbcl.so and the host-side (CPU) half of the API:
chunking, schedules, cost models, tuning tables. Everything here executes in
the product's C++ (bcl_core.cpp / bcl_tuner.cpp); Python only marshals."""
import ctypes as C
import enum
import math
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))


def lib_path() -> str:
    # BCL_LIB: load an alternative build (development experiments only)
    return os.environ.get("BCL_LIB") or os.path.join(_HERE, "libbcl.so")


class BclError(RuntimeError):
    """std::runtime_error family (BCL_ERR_RUNTIME)."""


class TableParseError(BclError):
    """tuner.hpp:76-83: carries the 1-based line number."""

    def __init__(self, msg, line):
        super().__init__(msg)
        self.line = line


class CudaError(BclError):
    pass


class DeviceTimeout(BclError):
    pass


class AggregateRankError(BclError):
    pass


class _Config(C.Structure):
    _fields_ = [("algorithm", C.c_int32), ("radix_k", C.c_int32), ("chunk_bytes", C.c_uint64)]


class _Chunk(C.Structure):
    _fields_ = [("chunk_id", C.c_uint32), ("offset_bytes", C.c_uint64), ("length_bytes", C.c_uint64)]


class _Event(C.Structure):
    _fields_ = [("kind", C.c_int32), ("peer", C.c_int32), ("chunk", C.c_uint32), ("group", C.c_uint32)]


class _Entry(C.Structure):
    _fields_ = [("n", C.c_int32), ("msg_min_bytes", C.c_uint64), ("msg_max_bytes", C.c_uint64),
                ("config", _Config), ("predicted_cost_s", C.c_double)]


class _Net(C.Structure):
    _fields_ = [("startup_s", C.c_double), ("link_Bps", C.c_double), ("staging_Bps", C.c_double),
                ("call_overhead_s", C.c_double)]


_COST_FN = C.CFUNCTYPE(C.c_double, C.POINTER(_Config), C.c_int, C.c_uint64, C.c_void_p)

_SIGS = {
    "bcl_last_error": (C.c_char_p, []),
    "bcl_last_error_line": (C.c_size_t, []),
    "bcl_version": (C.c_char_p, []),
    "bcl_make_chunks": (C.c_int, [C.c_uint64, C.c_uint64, C.POINTER(_Chunk), C.c_size_t, C.POINTER(C.c_size_t)]),
    "bcl_schedule_create": (C.c_int, [C.POINTER(_Config), C.c_int, C.c_int, C.c_uint64, C.POINTER(C.c_void_p)]),
    "bcl_schedule_destroy": (C.c_int, [C.c_void_p]),
    "bcl_schedule_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_uint64),
                                    C.POINTER(C.c_int), C.POINTER(C.c_size_t)]),
    "bcl_schedule_chunks": (C.c_int, [C.c_void_p, C.POINTER(_Chunk), C.c_size_t]),
    "bcl_schedule_rank_events": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(_Event), C.c_size_t, C.POINTER(C.c_size_t)]),
    "bcl_schedule_validate": (C.c_int, [C.c_void_p]),
    "bcl_schedule_text": (C.c_int, [C.c_void_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "bcl_model_cost": (C.c_int, [C.POINTER(_Config), C.c_int, C.c_uint64, C.c_double, C.c_double, C.c_double,
                                 C.POINTER(C.c_double)]),
    "bcl_tune_analytical": (C.c_int, [C.POINTER(C.c_int), C.c_size_t, C.POINTER(C.c_uint64), C.c_size_t,
                                      C.POINTER(_Config), C.c_size_t, C.POINTER(C.c_uint64), C.c_size_t,
                                      C.c_double, C.c_double, C.c_double, C.POINTER(C.c_void_p)]),
    "bcl_model_cost_ex": (C.c_int, [C.POINTER(_Config), C.c_int, C.c_uint64, C.POINTER(_Net), C.POINTER(C.c_double)]),
    "bcl_tune_analytical_ex": (C.c_int, [C.POINTER(C.c_int), C.c_size_t, C.POINTER(C.c_uint64), C.c_size_t,
                                         C.POINTER(_Config), C.c_size_t, C.POINTER(C.c_uint64), C.c_size_t,
                                         C.POINTER(_Net), C.POINTER(C.c_void_p)]),
    "bcl_tune_measured": (C.c_int, [C.POINTER(C.c_int), C.c_size_t, C.POINTER(C.c_uint64), C.c_size_t,
                                    C.POINTER(_Config), C.c_size_t, C.POINTER(C.c_uint64), C.c_size_t,
                                    _COST_FN, C.c_void_p, C.c_char_p, C.POINTER(C.c_void_p)]),
    "bcl_table_load": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "bcl_table_load_text": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "bcl_table_save": (C.c_int, [C.c_void_p, C.c_char_p]),
    "bcl_table_save_text": (C.c_int, [C.c_void_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "bcl_table_builtin": (C.c_int, [C.POINTER(C.c_void_p)]),
    "bcl_table_destroy": (C.c_int, [C.c_void_p]),
    "bcl_table_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_size_t)]),
    "bcl_table_entries": (C.c_int, [C.c_void_p, C.POINTER(_Entry), C.c_size_t]),
    "bcl_table_select": (C.c_int, [C.c_void_p, C.c_int, C.c_uint64, C.POINTER(_Config)]),
    "bcl_comm_init_all": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.c_double, C.POINTER(C.c_void_p)]),
    "bcl_comm_init_rank": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_size_t, C.c_double, C.POINTER(C.c_void_p)]),
    "bcl_comm_init_all_opts": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.c_char_p, C.POINTER(C.c_void_p)]),
    "bcl_comm_init_rank_opts": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_size_t, C.c_char_p, C.POINTER(C.c_void_p)]),
    "bcl_comm_export": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "bcl_comm_connect": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t]),
    "bcl_comm_destroy": (C.c_int, [C.c_void_p]),
    "bcl_comm_register_export": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t,
                                           C.POINTER(C.c_size_t)]),
    "bcl_comm_register_connect": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t]),
    "bcl_comm_protocol_caps": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                         C.POINTER(C.c_uint64)]),
    "bcl_comm_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                C.POINTER(C.c_int)]),
    "bcl_comm_set_table": (C.c_int, [C.c_void_p, C.c_void_p]),
    "bcl_comm_choose": (C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(_Config)]),
    "bcl_comm_set_protocol": (C.c_int, [C.c_void_p, C.c_int]),
    "bcl_group_start": (C.c_int, []),
    "bcl_group_end": (C.c_int, []),
    "bcl_comm_nvls": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "bcl_comm_path": (C.c_int, [C.c_void_p, C.POINTER(_Config), C.c_int, C.c_uint64, C.c_char_p, C.c_size_t,
                                C.POINTER(C.c_size_t)]),
    "bcl_comm_plan": (C.c_int, [C.c_void_p, C.POINTER(_Config), C.c_int, C.c_uint64, C.POINTER(C.c_int),
                                C.POINTER(C.c_uint64), C.POINTER(C.c_uint32), C.POINTER(C.c_int)]),
    "bcl_mem_alloc": (C.c_int, [C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]),
    "bcl_mem_reset": (C.c_int, [C.c_void_p]),
    "bcl_bcast": (C.c_int, [C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_void_p, C.POINTER(_Config), C.c_void_p]),
    "bcl_bcast_host": (C.c_int, [C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_void_p, C.POINTER(_Config),
                                 C.c_void_p]),
    "bcl_bcast_all": (C.c_int, [C.POINTER(C.c_void_p), C.c_size_t, C.c_int, C.c_int, C.POINTER(C.c_void_p),
                                C.c_int, C.POINTER(_Config), C.POINTER(C.c_void_p)]),
    "bcl_run_bcast": (C.c_int, [C.c_int, C.c_int, C.POINTER(C.c_void_p), C.c_uint64, C.POINTER(_Config),
                                C.POINTER(C.c_void_p), C.POINTER(C.c_double)]),
    "bcl_run_bcast_host": (C.c_int, [C.c_int, C.c_int, C.POINTER(C.c_void_p), C.c_uint64, C.POINTER(_Config),
                                     C.POINTER(C.c_void_p), C.POINTER(C.c_double)]),
    "bcl_barrier": (C.c_int, [C.c_void_p, C.c_void_p]),
    "bcl_barrier_all": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.POINTER(C.c_void_p)]),
    "bcl_comm_check": (C.c_int, [C.c_void_p, C.c_void_p]),
    "bcl_comm_set_provenance": (C.c_int, [C.c_void_p, C.c_void_p]),
    "bcl_comm_set_trace": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint32]),
    "bcl_comm_launches": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64)]),
}

_lib = None


def lib():
    """The loaded libbcl.so; raises ImportError when it was not built."""
    global _lib
    if _lib is None:
        path = lib_path()
        if not os.path.exists(path):
            raise ImportError(f"{path} is missing: build it with `make -C {_HERE}` (no CPU fallback exists)")
        l = C.CDLL(path)
        for name, (res, args) in _SIGS.items():
            try:
                f = getattr(l, name)
            except AttributeError:
                if os.environ.get("BCL_LIB"):  # an older experimental build: its missing entry points raise if called
                    continue
                raise
            f.restype = res
            f.argtypes = args
        _lib = l
    return _lib


def _check(status):
    if status == 0:
        return
    msg = lib().bcl_last_error().decode(errors="replace")
    if status == 1:
        raise ValueError(msg)  # std::invalid_argument
    if status == 3:
        raise IndexError(msg)  # std::out_of_range
    if status == 4:
        raise TableParseError(msg, lib().bcl_last_error_line())
    if status == 6:
        raise CudaError(msg)
    if status == 7:
        raise DeviceTimeout(msg)
    if status == 8:
        raise AggregateRankError(msg)
    if status == 5:
        raise OSError(msg)
    raise BclError(msg)


class Algorithm(enum.IntEnum):
    """core.hpp:27-34 (enum order is the tuner tie-break order)."""
    direct = 0
    chain = 1
    knomial = 2
    scatter_ring_allgather = 3
    chain_pipelined = 4
    knomial_staged = 5


ALGORITHMS = [a.name for a in Algorithm]

DTYPES = {"int8": 0, "uint8": 1, "int32": 2, "uint32": 3, "int64": 4, "uint64": 5,
          "float16": 6, "float32": 7, "float64": 8, "bfloat16": 9}


@dataclass(frozen=True)
class AlgorithmConfig:
    algorithm: Algorithm = Algorithm.chain
    radix_k: int = 0
    chunk_bytes: int = 0

    def _c(self):
        c = self.__dict__.get("_cached")  # (immutable: built once, passed by reference on every call)
        if c is None:
            c = _Config(int(self.algorithm), self.radix_k, self.chunk_bytes)
            object.__setattr__(self, "_cached", c)
        return c

    @staticmethod
    def _from(c):
        return AlgorithmConfig(Algorithm(c.algorithm), c.radix_k, c.chunk_bytes)

    @staticmethod
    def of(name, radix_k=0, chunk_bytes=0):
        return AlgorithmConfig(Algorithm[name], radix_k, chunk_bytes)


@dataclass(frozen=True)
class ChunkSpec:
    chunk_id: int
    offset_bytes: int
    length_bytes: int


@dataclass(frozen=True)
class Event:
    kind: str  # "send" | "recv"
    peer: int
    chunk: int
    group: int = 0


@dataclass
class Schedule:
    n_ranks: int
    root: int
    message_bytes: int
    prologue: int
    chunks: List[ChunkSpec]
    per_rank_ops: List[List[Event]]
    _handle: Optional[int] = field(default=None, repr=False, compare=False)


def make_chunks(message_bytes: int, chunk_bytes: int) -> List[ChunkSpec]:
    n = C.c_size_t()
    _check(lib().bcl_make_chunks(message_bytes, chunk_bytes, None, 0, C.byref(n)))
    arr = (_Chunk * n.value)()
    _check(lib().bcl_make_chunks(message_bytes, chunk_bytes, arr, n.value, C.byref(n)))
    return [ChunkSpec(c.chunk_id, c.offset_bytes, c.length_bytes) for c in arr]


def _schedule(cfg: AlgorithmConfig, n: int, root: int, m: int) -> Schedule:
    h = C.c_void_p()
    cc = cfg._c()
    _check(lib().bcl_schedule_create(C.byref(cc), n, root, m, C.byref(h)))
    try:
        nn, rr, mm, pro, nch = C.c_int(), C.c_int(), C.c_uint64(), C.c_int(), C.c_size_t()
        _check(lib().bcl_schedule_info(h, C.byref(nn), C.byref(rr), C.byref(mm), C.byref(pro), C.byref(nch)))
        chunks = (_Chunk * max(nch.value, 1))()
        _check(lib().bcl_schedule_chunks(h, chunks, nch.value))
        ops = []
        for r in range(nn.value):
            cnt = C.c_size_t()
            _check(lib().bcl_schedule_rank_events(h, r, None, 0, C.byref(cnt)))
            ev = (_Event * max(cnt.value, 1))()
            _check(lib().bcl_schedule_rank_events(h, r, ev, cnt.value, C.byref(cnt)))
            ops.append([Event("send" if e.kind == 0 else "recv", e.peer, e.chunk, e.group)
                        for e in ev[:cnt.value]])
        return Schedule(nn.value, rr.value, mm.value, pro.value,
                        [ChunkSpec(c.chunk_id, c.offset_bytes, c.length_bytes) for c in chunks[:nch.value]], ops)
    finally:
        lib().bcl_schedule_destroy(h)


def make_schedule(config: AlgorithmConfig, n: int, root: int, message_bytes: int) -> Schedule:
    return _schedule(config, n, root, message_bytes)


def schedule_direct(n, root, m):
    return _schedule(AlgorithmConfig(Algorithm.direct), n, root, m)


def schedule_chain(n, root, m):
    return _schedule(AlgorithmConfig(Algorithm.chain), n, root, m)


def schedule_knomial(n, radix_k, root, m):
    return _schedule(AlgorithmConfig(Algorithm.knomial, radix_k), n, root, m)


def schedule_knomial_staged(n, radix_k, root, m):
    return _schedule(AlgorithmConfig(Algorithm.knomial_staged, radix_k), n, root, m)


def schedule_scatter_ring_allgather(n, root, m):
    return _schedule(AlgorithmConfig(Algorithm.scatter_ring_allgather), n, root, m)


def schedule_chain_pipelined(n, root, m, chunk_bytes):
    return _schedule(AlgorithmConfig(Algorithm.chain_pipelined, 0, chunk_bytes), n, root, m)


def validate_schedule(config: AlgorithmConfig, n: int, root: int, m: int) -> Optional[str]:
    """validate_schedule(make_schedule(...)) -> None or the violation text."""
    h = C.c_void_p()
    cc = config._c()
    _check(lib().bcl_schedule_create(C.byref(cc), n, root, m, C.byref(h)))
    try:
        st = lib().bcl_schedule_validate(h)
        return None if st == 0 else lib().bcl_last_error().decode()
    finally:
        lib().bcl_schedule_destroy(h)


def to_text(config: AlgorithmConfig, n: int, root: int, m: int) -> str:
    h = C.c_void_p()
    cc = config._c()
    _check(lib().bcl_schedule_create(C.byref(cc), n, root, m, C.byref(h)))
    try:
        ln = C.c_size_t()
        _check(lib().bcl_schedule_text(h, None, 0, C.byref(ln)))
        buf = C.create_string_buffer(ln.value)
        _check(lib().bcl_schedule_text(h, buf, ln.value, C.byref(ln)))
        return buf.value.decode()
    finally:
        lib().bcl_schedule_destroy(h)


def cost_for(config: AlgorithmConfig, n: int, m: int, startup_s=1e-6, link_Bps=1e9, staging_Bps=1e10,
             call_overhead_s=0.0) -> float:
    """models.cpp:106-124; call_overhead_s = the B200 per-call constant a0 (0: the reference model)."""
    out = C.c_double()
    cc = config._c()
    if call_overhead_s:
        net = _Net(startup_s, link_Bps, staging_Bps, call_overhead_s)
        _check(lib().bcl_model_cost_ex(C.byref(cc), n, m, C.byref(net), C.byref(out)))
    else:
        _check(lib().bcl_model_cost(C.byref(cc), n, m, startup_s, link_Bps, staging_Bps, C.byref(out)))
    return out.value


@dataclass(frozen=True)
class TuningEntry:
    n: int
    msg_min_bytes: int
    msg_max_bytes: int
    config: AlgorithmConfig
    predicted_cost_s: float


class TuningTable:
    """Owns a C++ TuningTable (tuner.hpp:31-38)."""

    def __init__(self, handle):
        self._h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.bcl_table_destroy(h)
            self._h = None

    @property
    def oracle(self) -> str:
        o = C.c_int()
        _check(lib().bcl_table_info(self._h, C.byref(o), None))
        return ["analytical", "simulated", "measured"][o.value]

    @property
    def entries(self) -> List[TuningEntry]:
        n = C.c_size_t()
        _check(lib().bcl_table_info(self._h, None, C.byref(n)))
        arr = (_Entry * max(n.value, 1))()
        _check(lib().bcl_table_entries(self._h, arr, n.value))
        return [TuningEntry(e.n, e.msg_min_bytes, e.msg_max_bytes, AlgorithmConfig._from(e.config),
                            e.predicted_cost_s) for e in arr[:n.value]]

    def select(self, n: int, message_bytes: int) -> AlgorithmConfig:
        return select(self, n, message_bytes)

    def text(self) -> str:
        return save_table_text(self)

    def __eq__(self, other):
        return isinstance(other, TuningTable) and self.oracle == other.oracle and self.entries == other.entries


def _cands(candidates: Sequence[AlgorithmConfig]):
    return (_Config * max(len(candidates), 1))(*[c._c() for c in candidates])


def tune(n_list, msg_sizes, candidates, chunk_candidates, startup_s=1e-6, link_Bps=1e9,
         staging_Bps=1e10, call_overhead_s=0.0) -> TuningTable:
    """tuner.hpp:64-68 with the analytical oracle (plus the B200 per-call
    constant a0 when call_overhead_s > 0)."""
    h = C.c_void_p()
    nl = (C.c_int * max(len(n_list), 1))(*n_list)
    sz = (C.c_uint64 * max(len(msg_sizes), 1))(*msg_sizes)
    ch = (C.c_uint64 * max(len(chunk_candidates), 1))(*chunk_candidates)
    if call_overhead_s:
        net = _Net(startup_s, link_Bps, staging_Bps, call_overhead_s)
        _check(lib().bcl_tune_analytical_ex(nl, len(n_list), sz, len(msg_sizes), _cands(candidates),
                                            len(candidates), ch, len(chunk_candidates), C.byref(net), C.byref(h)))
    else:
        _check(lib().bcl_tune_analytical(nl, len(n_list), sz, len(msg_sizes), _cands(candidates), len(candidates),
                                         ch, len(chunk_candidates), startup_s, link_Bps, staging_Bps, C.byref(h)))
    return TuningTable(h)


def tune_measured(n_list, msg_sizes, candidates, chunk_candidates, cost, provenance="") -> TuningTable:
    """Same brute force with cost(config, n, bytes) -> seconds supplied by a
    measurement (the B200 Measured oracle)."""
    failure = []

    def _cb(cfg_p, n, m, _user):
        try:
            return float(cost(AlgorithmConfig._from(cfg_p.contents), n, m))
        except Exception as e:  # noqa: BLE001 - surfaces as BCL_ERR_RUNTIME, re-raised below
            failure.append(e)
            return math.nan
    cb = _COST_FN(_cb)
    h = C.c_void_p()
    nl = (C.c_int * max(len(n_list), 1))(*n_list)
    sz = (C.c_uint64 * max(len(msg_sizes), 1))(*msg_sizes)
    ch = (C.c_uint64 * max(len(chunk_candidates), 1))(*chunk_candidates)
    try:
        _check(lib().bcl_tune_measured(nl, len(n_list), sz, len(msg_sizes), _cands(candidates), len(candidates),
                                       ch, len(chunk_candidates), cb, None, provenance.encode(), C.byref(h)))
    except BclError as e:
        if failure:
            raise failure[0] from e
        raise
    return TuningTable(h)


def select(table: TuningTable, n: int, message_bytes: int) -> AlgorithmConfig:
    out = _Config()
    _check(lib().bcl_table_select(table._h, n, message_bytes, C.byref(out)))
    return AlgorithmConfig._from(out)


def load_table(path: str) -> TuningTable:
    h = C.c_void_p()
    _check(lib().bcl_table_load(os.fsencode(path), C.byref(h)))
    return TuningTable(h)


def load_table_text(text: str) -> TuningTable:
    h = C.c_void_p()
    _check(lib().bcl_table_load_text(text.encode(), C.byref(h)))
    return TuningTable(h)


def save_table(table: TuningTable, path: str) -> None:
    _check(lib().bcl_table_save(table._h, os.fsencode(path)))


def save_table_text(table: TuningTable) -> str:
    ln = C.c_size_t()
    _check(lib().bcl_table_save_text(table._h, None, 0, C.byref(ln)))
    buf = C.create_string_buffer(ln.value)
    _check(lib().bcl_table_save_text(table._h, buf, ln.value, C.byref(ln)))
    return buf.value.decode()


def builtin_table() -> TuningTable:
    h = C.c_void_p()
    _check(lib().bcl_table_builtin(C.byref(h)))
    return TuningTable(h)
