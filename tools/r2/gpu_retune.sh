# Re-derive the measured tables with the round-2 kernels (LL128 ring).
set -x
N=$(nvidia-smi -L | wc -l)
OUT=gpurun_out/r2tune_n$N
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 2400 $TR --master-port 29540 tools/tune_b200.py --out $OUT/b200_measured_n$N.csv --raw $OUT/raw$N.csv > $OUT/tune.log 2>&1
echo "tune rc=$?"; tail -30 $OUT/tune.log
