#!/bin/bash
# LL128 direct in its own landing areas: multi-GPU suites, soak, A/B, configs 4/5 grouped.
out=gpurun_out/d128c; mkdir -p $out
(cd paper_1707_09414_b200 && make -s >/dev/null)
timeout 700 python -m pytest tests/test_multigpu.py tests/test_nvls.py -x -q 2>&1 | tail -3 | tee $out/pytest4.txt
timeout 400 python tools/r2/soak.py 800 13 2>&1 | tail -3 | tee $out/soak4.txt
SIZES=65536,131072,262144,524288,1048576,2097152 ITERS=15 B2B=8 ALGO=direct VARIANTS="auto;auto:ll128_direct_min=0" \
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29614 \
  tools/r2/proto_ab.py 2>&1 | grep "N=" | tee -a $out/ab.txt
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
p=29760
for wl in resnet50; do
  for f in "" "--fused" "--fused --graph"; do
    p=$((p+1))
    tag=${wl}$(echo $f | tr -d ' -')
    timeout 150 $TR --nproc-per-node 4 --master-port $p bench.py --gpus 4 --workload $wl $f --steps 10 --warmup 3 > $out/$tag.json 2> $out/$tag.err
    echo "$wl [$f] rc=$? $(tail -1 $out/$tag.json | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["nccl_ms"], d["gpu_launches"])' 2>&1)"
  done
done
