"""B200-native pipelined-chain broadcast (arXiv:1707.09414 hot path).

Python mirror of the reference's public surface (bcastlab, /root/reference/proj)
over the C-ABI of libbcl.so (include/bcl.h). Same names, argument meaning and
error behaviour as the reference:

  make_chunks, make_schedule, schedule_* , validate_schedule, to_text  (core/schedules)
  cost_for, tune, select, load_table, save_table, TableParseError      (models/tuner)
  Comm.local / Comm.rank, bcast, bcast_all, run_bcast                  (runtime)

There is no CPU fallback: importing this package without the built CUDA
library raises ImportError (build with ``make -C paper_1707_09414_b200`` or
``python -c "import __graft_entry__ as g; g.build()"``).
"""
from ._lib import (  # noqa: F401
    ALGORITHMS, Algorithm, AlgorithmConfig, ChunkSpec, Event, Schedule, TuningEntry,
    TuningTable, TableParseError, DeviceTimeout, AggregateRankError, CudaError,
    BclError, lib, lib_path, make_chunks, make_schedule, schedule_direct, schedule_chain,
    schedule_knomial, schedule_knomial_staged, schedule_scatter_ring_allgather,
    schedule_chain_pipelined, validate_schedule, to_text, cost_for, tune, tune_measured,
    select, load_table, load_table_text, save_table, save_table_text, builtin_table,
    DTYPES,
)
from .comm import Comm, run_bcast, run_bcast_host, bcast_all, barrier_all, DevicePtr, group  # noqa: F401
