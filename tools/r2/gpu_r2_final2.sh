# Round-2 final tree (LL128 direct lines) on a 4-GPU box: full GPU suite, N=4 and N=2 benches (sweep + NVLS
# column), configs 4/5 per tensor eager / graph / grouped at N=4.
N=$(nvidia-smi -L | wc -l)
OUT=gpurun_out/r2final2
mkdir -p $OUT
(cd paper_1707_09414_b200 && make -s >/dev/null)
timeout 1200 python -m pytest tests -q -m gpu > $OUT/pytest_gpu_${N}gpu.log 2>&1
echo "pytest rc=$? $(tail -1 $OUT/pytest_gpu_${N}gpu.log)"
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node $N --master-port 29561 bench.py --gpus $N --csv $OUT/bench_sweep_n$N.csv > $OUT/bench_n$N.json 2> $OUT/bench_n$N.err
echo "bench n$N rc=$?"
CUDA_VISIBLE_DEVICES=0,1 timeout 900 $TR --nproc-per-node 2 --master-port 29562 bench.py --gpus 2 --csv $OUT/bench_sweep_n2.csv > $OUT/bench_n2.json 2> $OUT/bench_n2.err
echo "bench n2 rc=$?"
p=29750
for wl in resnet50 vgg16; do
  for f in "" "--graph" "--fused --graph"; do
    p=$((p+1))
    tag=${wl}$(echo $f | tr -d ' -')
    timeout 150 $TR --nproc-per-node $N --master-port $p bench.py --gpus $N --workload $wl $f --steps 10 --warmup 3 > $OUT/$tag.json 2> $OUT/$tag.err
    echo "$wl [$f] rc=$? $(tail -1 $OUT/$tag.json | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["nccl_ms"], d["gpu_launches"])' 2>&1)"
  done
done
