# N=4 (or N = visible GPUs): bench with the NVLS column, then re-tune with NVLS available.
set -x
N=$(nvidia-smi -L | wc -l)
OUT=gpurun_out/nvls_n$N
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 900 $TR --master-port 29541 bench.py --gpus $N --steps 10 --warmup 3 > $OUT/bench_n$N.json 2> $OUT/bench.err
echo "bench rc=$?"
timeout 2400 $TR --master-port 29542 tools/tune_b200.py --out $OUT/b200_measured_n$N.csv --raw $OUT/raw$N.csv > $OUT/tune.log 2>&1
echo "tune rc=$?"; tail -5 $OUT/tune.log
