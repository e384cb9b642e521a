# Multi-GPU pass (gpurun --gpus N): parity across GPUs, the writer-fence
# scope A/B on the pull path, a lane timeline, and the full bench line.
set -x
N=$(nvidia-smi -L | wc -l)
OUT=gpurun_out/r2m_n$N
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
if [ -z "$SKIP_PYTEST" ]; then
  timeout 900 python -m pytest tests/test_multigpu.py -x -q > $OUT/pytest_multi.log 2>&1; echo "pytest rc=$?"
  tail -3 $OUT/pytest_multi.log
fi
for wf in 2 1; do
  for sz in 67108864 1073741824; do
    BCL_PROTOCOL=1 BCL_WRITER_FENCE=$wf timeout 300 $TR --master-port $((29500+wf)) bench.py --gpus $N --steps 20 --warmup 5 --no-sweep --bytes $sz > $OUT/bench_pull_wf${wf}_$sz.json 2> $OUT/bench_pull_wf${wf}_$sz.err
    echo "wf=$wf sz=$sz rc=$?"; grep -o '"value": [0-9.]*\|"latency_us": {[^}]*}' $OUT/bench_pull_wf${wf}_$sz.json
  done
done
TRACE_BYTES=67108864 TRACE_CHUNK=65536 TRACE_ITERS=6 timeout 300 $TR --master-port 29520 tools/trace_mp.py > $OUT/trace_64m.log 2>&1; echo "trace rc=$?"; grep -v "^\[\|NCCL\|\*\*\*\|OMP" $OUT/trace_64m.log | tail -8
timeout 1500 $TR --master-port 29510 bench.py --gpus $N --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err
echo "bench rc=$?"
head -c 3000 $OUT/bench.json
