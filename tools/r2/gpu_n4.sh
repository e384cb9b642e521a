# 4-GPU pass: every GPU test, NVML counter probe, NVLS probe v2, e2e probe, N=4 bench.
set -x
N=$(nvidia-smi -L | wc -l)
OUT=gpurun_out/r2_n$N
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke.log
timeout 120 python tools/r2/nvml_probe.py > $OUT/nvml_probe.log 2>&1; echo "nvml rc=$?"; tail -9 $OUT/nvml_probe.log
timeout 300 tools/r2/nvls_probe2 $N 16777216 67108864 268435456 1073741824 > $OUT/nvls_probe2.log 2>&1; echo "nvls rc=$?"; cat $OUT/nvls_probe2.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/r2/e2e_probe2.py > $OUT/e2e_probe2.log 2>&1; echo "e2e rc=$?"; cat $OUT/e2e_probe2.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 1500 $TR --master-port 29510 bench.py --gpus $N --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err
echo "bench rc=$?"
head -c 2500 $OUT/bench.json
