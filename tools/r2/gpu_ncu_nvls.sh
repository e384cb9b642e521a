# ncu of the NVLS kernels (root = multicast writer on GPU 0, receiver on GPU 1):
# kernel replay cannot save/restore multicast-bound memory, so application replay.
set -x
OUT=gpurun_out/r2_ncu
mkdir -p $OUT
export CUDA_VISIBLE_DEVICES=0,1
NVM="nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
timeout 900 ncu --replay-mode application --metrics $NVM --section SpeedOfLight --section WarpStateStats --clock-control none -k regex:nvls_kernel -c 2 -o $OUT/ncu_nvls python tools/r2/ncu_xgpu.py nvls 33554432 > $OUT/ncu_nvls.log 2>&1
echo "ncu nvls rc=$?"; tail -3 $OUT/ncu_nvls.log
