# 4-GPU pass: N=4 bench (LL128 ring with cached credits), emulated n=8 table
# (2 ranks per GPU), reference CPU sweep on this host.
set -x
N=$(nvidia-smi -L | wc -l)
OUT=gpurun_out/r2b_n$N
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 1500 $TR --master-port 29510 bench.py --gpus $N --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err
echo "bench rc=$?"; head -c 1200 $OUT/bench.json
timeout 1500 python tools/tune_local.py --devices 0,0,1,1,2,2,3,3 --out $OUT/b200_emulated_n8.csv --max 268435456 > $OUT/tune_local.log 2>&1
echo "tune_local rc=$?"; tail -25 $OUT/tune_local.log
timeout 900 python tools/cpu_sweep.py --ranks 2,4,8 > $OUT/cpu_sweep.json 2> $OUT/cpu_sweep.err; echo "cpu sweep rc=$?"; tail -3 $OUT/cpu_sweep.err
