# ncu evidence after the round-2 kernel changes: N=1 launch list + full capture
# of local_chain_kernel (GPU 0), NVLS kernels across two GPUs (one process).
set -x
OUT=gpurun_out/r2_ncu
mkdir -p $OUT
export CUDA_VISIBLE_DEVICES=0
timeout 600 python bench.py --steps 3 --warmup 3 --cpu-iters 1 > $OUT/plain_small.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 --cpu-iters 1 > $OUT/ncu_launches.log 2>&1
echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:local_chain_kernel -s 4 -c 1 -o $OUT/prof_local_chain python bench.py --steps 3 --warmup 3 --cpu-iters 1 > $OUT/ncu_full.log 2>&1
echo "ncu full rc=$?"; tail -2 $OUT/ncu_full.log
export CUDA_VISIBLE_DEVICES=0,1
NVM="nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
timeout 120 python tools/r2/ncu_xgpu.py nvls 33554432 > $OUT/xgpu_nvls_plain.log 2>&1 && \
timeout 600 ncu --set full --metrics $NVM --clock-control none --import-source on -k regex:nvls_kernel -c 2 -o $OUT/ncu_nvls python tools/r2/ncu_xgpu.py nvls 33554432 > $OUT/ncu_nvls.log 2>&1
echo "ncu nvls rc=$?"; tail -3 $OUT/ncu_nvls.log
