# Round-2 evidence on a 4-GPU box: full GPU suite, then N=4 and N=2 benches (sweep + NVLS column).
N=$(nvidia-smi -L | wc -l)
OUT=gpurun_out/r2final
mkdir -p $OUT
timeout 1200 python -m pytest tests -q -m gpu > $OUT/pytest_gpu_${N}gpu.log 2>&1
echo "pytest rc=$? $(tail -1 $OUT/pytest_gpu_${N}gpu.log)"
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node $N --master-port 29561 bench.py --gpus $N --csv $OUT/bench_sweep_n$N.csv > $OUT/bench_n$N.json 2> $OUT/bench_n$N.err
echo "bench n$N rc=$?"
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR --nproc-per-node 2 --master-port 29562 bench.py --gpus 2 --csv $OUT/bench_sweep_n2.csv > $OUT/bench_n2.json 2> $OUT/bench_n2.err
echo "bench n2 rc=$?"
