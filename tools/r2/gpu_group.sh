# Multi-GPU suite (incl. group fusion across GPUs and NVLS) + configs 4/5 grouped vs per tensor.
N=$(nvidia-smi -L | wc -l)
OUT=gpurun_out/group_n$N
mkdir -p $OUT
timeout 900 python -m pytest tests/test_multigpu.py tests/test_nvls.py -q -m gpu > $OUT/pytest_multi.log 2>&1
echo "pytest rc=$? $(tail -1 $OUT/pytest_multi.log)"
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
p=29580
for wl in resnet50 lenet vgg16 alexnet; do
  for f in "" "--fused"; do
    p=$((p+1))
    timeout 600 $TR --master-port $p bench.py --gpus $N --workload $wl $f --steps 10 --warmup 3 > $OUT/${wl}${f// /}.json 2> $OUT/${wl}${f// /}.err
    echo "$wl $f rc=$? $(tail -1 $OUT/${wl}${f// /}.json | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["nccl_ms"], d["gpu_launches"])' 2>&1)"
  done
done
