# Host-path trims (shared plans, lean Python bcast): multi-GPU suite, host enqueue cost per call, configs 4/5 eager.
OUT=gpurun_out/hostpath; mkdir -p $OUT
(cd paper_1707_09414_b200 && make -s >/dev/null)
timeout 700 python -m pytest tests/test_multigpu.py -x -q 2>&1 | tail -2 | tee $OUT/pytest4.txt
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
timeout 300 $TR --master-port 29740 tools/r2/hostbound_probe.py 2>&1 | grep "N=" | tee $OUT/hostbound_n4.txt
p=29750
for wl in resnet50 vgg16; do
  for f in "" "--graph"; do
    p=$((p+1)); tag=${wl}$(echo $f | tr -d ' -')
    timeout 150 $TR --master-port $p bench.py --gpus 4 --workload $wl $f --steps 10 --warmup 3 > $OUT/$tag.json 2> $OUT/$tag.err
    echo "$wl [$f] rc=$? $(tail -1 $OUT/$tag.json | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["nccl_ms"], d["gpu_launches"])' 2>&1)"
  done
done
