#!/bin/bash
# Fused LL128 direct lines in groups: 1-GPU group/LL128 tests (first GPU only), multi-GPU suites, soak,
# configs 4/5 grouped at N=4.
out=gpurun_out/d128d; mkdir -p $out
(cd paper_1707_09414_b200 && make -s >/dev/null)
CUDA_VISIBLE_DEVICES=0 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "group or ll128 or graph" 2>&1 | tail -3 | tee $out/pytest1.txt
timeout 700 python -m pytest tests/test_multigpu.py tests/test_nvls.py -x -q 2>&1 | tail -3 | tee $out/pytest4.txt
timeout 400 python tools/r2/soak.py 800 17 2>&1 | tail -3 | tee $out/soak4.txt
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
p=29770
for wl in resnet50 vgg16 alexnet; do
  for f in "--fused" "--fused --graph"; do
    p=$((p+1))
    tag=${wl}$(echo $f | tr -d ' -')
    timeout 150 $TR --nproc-per-node 4 --master-port $p bench.py --gpus 4 --workload $wl $f --steps 10 --warmup 3 > $out/$tag.json 2> $out/$tag.err
    echo "$wl [$f] rc=$? $(tail -1 $out/$tag.json | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["nccl_ms"], d["gpu_launches"])' 2>&1)"
  done
done
