# Configs 4/5 per tensor: eager vs CUDA-graph replay vs grouped (+graph), ours and NCCL, N GPUs.
N=$(nvidia-smi -L | wc -l)
OUT=gpurun_out/graphs_n$N
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
p=29750
for wl in resnet50 lenet vgg16 alexnet; do
  for f in "" "--graph" "--fused" "--fused --graph"; do
    p=$((p+1))
    tag=${wl}$(echo $f | tr -d ' -')
    timeout 150 $TR --master-port $p bench.py --gpus $N --workload $wl $f --steps 10 --warmup 3 > $OUT/$tag.json 2> $OUT/$tag.err
    echo "$wl [$f] rc=$? $(tail -1 $OUT/$tag.json | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["nccl_ms"], d["gpu_launches"])' 2>&1)"
  done
done
