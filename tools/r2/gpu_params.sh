# Configs 4/5 (layer-wise parameter broadcast) on N GPUs, per tensor and bucketed.
N=$(nvidia-smi -L | wc -l)
OUT=gpurun_out/params_n$N
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
p=29570
for wl in vgg16 alexnet resnet50 lenet; do
  for b in 0 4194304; do
    p=$((p+1))
    timeout 600 $TR --master-port $p bench.py --gpus $N --workload $wl --bucket $b --steps 10 --warmup 3 > $OUT/${wl}_b$b.json 2> $OUT/${wl}_b$b.err
    echo "$wl bucket $b rc=$? $(tail -1 $OUT/${wl}_b$b.json | cut -c1-200)"
  done
done
