#!/bin/bash
# One gpurun call: GPU tests, N=1 bench, launch list and one ncu --set full
# capture of the broadcast kernel (same command line run plain first).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err
CMD="python bench.py --steps 2 --warmup 3 --cpu-iters 1"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n1.csv $CMD > gpurun_out/ncu_launch.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:bcast_kernel -s 3 -c 1 -o gpurun_out/prof_n1 $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full.log
