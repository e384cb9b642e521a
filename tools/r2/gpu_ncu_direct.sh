# ncu of the direct schedule's line kernels at 2 MiB, N=2 in one process: application replay (kernel replay
# fails on these launches), SpeedOfLight + NVLink/DRAM counters, root (device 0) and receiver (device 1).
OUT=gpurun_out/r2final3
mkdir -p $OUT
(cd paper_1707_09414_b200 && make -s >/dev/null)
NVM="nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
for mode in direct128 direct_ll; do
  kern=$( [ $mode = direct128 ] && echo ll128_direct_kernel || echo ll_kernel )
  timeout 900 ncu --replay-mode application --metrics $NVM --section SpeedOfLight --section WarpStateStats --clock-control none \
    -k regex:$kern -c 2 -o $OUT/ncu_$mode python tools/r2/ncu_xgpu.py $mode 2097152 > $OUT/ncu_$mode.log 2>&1
  echo "ncu $mode rc=$?"
  ncu -i $OUT/ncu_$mode.ncu-rep --page details > $OUT/ncu_${mode}_details.txt 2>&1
done
