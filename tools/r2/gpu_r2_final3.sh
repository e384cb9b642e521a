# Round-2 final tree on a 4-GPU box: full GPU suite, N=4 / N=2 benches (sweeps + NVLS column), configs 4/5 at N=4
# (eager / graph / grouped / grouped+graph), ncu of the LL128 direct kernels vs 16-byte LL lines at 2 MiB (N=2,
# one process), a 2000-step soak.
N=$(nvidia-smi -L | wc -l)
OUT=gpurun_out/r2final3
mkdir -p $OUT
(cd paper_1707_09414_b200 && make -s >/dev/null)
timeout 1200 python -m pytest tests -q -m gpu > $OUT/pytest_gpu_${N}gpu.log 2>&1
echo "pytest rc=$? $(tail -1 $OUT/pytest_gpu_${N}gpu.log)"
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node $N --master-port 29561 bench.py --gpus $N --csv $OUT/bench_sweep_n$N.csv > $OUT/bench_n$N.json 2> $OUT/bench_n$N.err
echo "bench n$N rc=$?"
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR --nproc-per-node 2 --master-port 29562 bench.py --gpus 2 --csv $OUT/bench_sweep_n2.csv > $OUT/bench_n2.json 2> $OUT/bench_n2.err
echo "bench n2 rc=$?"
p=29780
for wl in resnet50 vgg16 alexnet lenet; do
  for f in "" "--graph" "--fused" "--fused --graph"; do
    p=$((p+1))
    tag=${wl}$(echo $f | tr -d ' -')
    timeout 150 $TR --nproc-per-node $N --master-port $p bench.py --gpus $N --workload $wl $f --steps 10 --warmup 3 > $OUT/$tag.json 2> $OUT/$tag.err
    echo "$wl [$f] rc=$? $(tail -1 $OUT/$tag.json | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["nccl_ms"], d["gpu_launches"])' 2>&1)"
  done
done
NVM="nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"
for mode in direct128 direct_ll; do
  kern=$( [ $mode = direct128 ] && echo ll128_direct_kernel || echo ll_kernel )
  timeout 120 python tools/r2/ncu_xgpu.py $mode 2097152 > $OUT/xgpu_${mode}_plain.log 2>&1 && \
  timeout 600 ncu --set full --metrics $NVM --clock-control none --import-source on -k regex:$kern -c 2 -o $OUT/ncu_$mode \
    python tools/r2/ncu_xgpu.py $mode 2097152 > $OUT/ncu_$mode.log 2>&1
  echo "ncu $mode rc=$?"
  ncu -i $OUT/ncu_$mode.ncu-rep --page details --section SpeedOfLight --metrics $NVM > $OUT/ncu_${mode}_details.txt 2>&1
done
timeout 900 python tools/r2/soak.py 2000 23 2>&1 | tail -2 | tee $OUT/soak4.log
