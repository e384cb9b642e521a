#!/bin/bash
# Re-derive the measured tables (N=4, N=2) with raw dumps (+ protocol rules),
# after the full GPU test suite.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/retune2; rm -f gpurun_out/retune2/*
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/retune2/tests.log 2>&1; echo "rc=$?" >> gpurun_out/retune2/tests.log
for N in 4 2; do
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 3020$N tools/tune_b200.py --out gpurun_out/retune2/t$N.csv --raw gpurun_out/retune2/raw$N.csv > gpurun_out/retune2/tune$N.log 2>&1
done
