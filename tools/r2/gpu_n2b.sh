# 2-GPU pass: multi-GPU parity (registration), ncu of the cross-GPU kernels
# (single process driving both GPUs, see tools/r2/ncu_xgpu.py), e2e probe, N=2 bench.
set -x
N=$(nvidia-smi -L | wc -l)
OUT=gpurun_out/r2b_n$N
mkdir -p $OUT
timeout 900 python -m pytest tests/test_multigpu.py -x -q > $OUT/pytest_multi.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_multi.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python tools/r2/e2e_probe3.py > $OUT/e2e_probe3.log 2>&1; echo "e2e rc=$?"; cat $OUT/e2e_probe3.log
NVM="nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
timeout 120 python tools/r2/ncu_xgpu.py pull 67108864 > $OUT/xgpu_pull_plain.log 2>&1 && \
timeout 600 ncu --devices 1 --set full --metrics $NVM --clock-control none --import-source on -k regex:bcast_kernel -c 1 -o $OUT/ncu_pull_rx python tools/r2/ncu_xgpu.py pull 67108864 > $OUT/ncu_pull.log 2>&1
echo "ncu pull rc=$?"; tail -3 $OUT/ncu_pull.log
timeout 120 python tools/r2/ncu_xgpu.py ll128 33554432 > $OUT/xgpu_ll128_plain.log 2>&1 && \
timeout 600 ncu --set full --metrics $NVM --clock-control none --import-source on -k regex:ll128_kernel -c 2 -o $OUT/ncu_ll128 python tools/r2/ncu_xgpu.py ll128 33554432 > $OUT/ncu_ll128.log 2>&1
echo "ncu ll128 rc=$?"; tail -3 $OUT/ncu_ll128.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 1500 $TR --master-port 29510 bench.py --gpus $N --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err
echo "bench rc=$?"
head -c 1500 $OUT/bench.json
