# Final tree, 2-GPU box: ncu of the direct schedule's line kernels (PDL off: ncu cannot replay a programmatic-
# dependent launch), then on GPU 0 alone the 1-GPU suite, smoke() and the N=1 bench line.
OUT=gpurun_out/r2final3
mkdir -p $OUT
(cd paper_1707_09414_b200 && make -s >/dev/null)
NVM="nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
for mode in direct128 direct_ll; do
  kern=$( [ $mode = direct128 ] && echo ll128_direct_kernel || echo ll_kernel )
  BCL_PDL=0 timeout 600 ncu --set full --metrics $NVM --clock-control none --import-source on -k regex:$kern -c 2 -o $OUT/ncu_$mode \
    python tools/r2/ncu_xgpu.py $mode 2097152 > $OUT/ncu_$mode.log 2>&1
  echo "ncu $mode rc=$?"
  ncu -i $OUT/ncu_$mode.ncu-rep --page details --section SpeedOfLight --metrics $NVM > $OUT/ncu_${mode}_details.txt 2>&1
done
export CUDA_VISIBLE_DEVICES=0
timeout 900 python -m pytest tests -q -m gpu > $OUT/pytest_gpu_1gpu.log 2>&1
echo "pytest 1gpu rc=$? $(tail -1 $OUT/pytest_gpu_1gpu.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_1gpu.log 2>&1
echo "smoke rc=$? $(tail -1 $OUT/smoke_1gpu.log)"
timeout 600 python bench.py > $OUT/bench_n1.json 2> $OUT/bench_n1.err
echo "bench n1 rc=$? $(tail -1 $OUT/bench_n1.json | cut -c1-300)"
