#!/bin/bash
# Re-derive the measured tables (N=4, N=2) with raw dumps, one device timeline
# in the reference trace schema, and an N=1 bench regression check.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/retune
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/retune/bench_n1.json 2> gpurun_out/retune/bench_n1.err
for N in 4 2; do
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 3020$N tools/tune_b200.py --out gpurun_out/retune/t$N.csv --raw gpurun_out/retune/raw$N.csv > gpurun_out/retune/tune$N.log 2>&1
done
TRACE_BYTES=67108864 TRACE_CHUNK=524288 TRACE_CSV=gpurun_out/retune/trace_n4_64m.csv timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 30209 tools/trace_mp.py > gpurun_out/retune/trace.log 2>&1
