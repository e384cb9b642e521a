#!/bin/bash
# Layer-wise parameter broadcast workloads (configs 4/5) at N=2 and N=4.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/params
for N in 2 4; do for W in vgg16 alexnet resnet50 lenet; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2980$N bench.py --gpus $N --workload $W --steps 10 --warmup 3 > gpurun_out/params/${W}_n$N.json 2> gpurun_out/params/${W}_n$N.err
done; done
