# N=4 host-buffer e2e under transport / piece variants (bench --no-sweep), to find what keeps it at 2x its DMA floor.
OUT=gpurun_out/e2en4; mkdir -p $OUT
(cd paper_1707_09414_b200 && make -s >/dev/null)
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 4"
p=29700
for v in "base:" "pull:BCL_PROTOCOL=1" "piece4m:BCL_HOST_PIECE=4194304" "piece64m:BCL_HOST_PIECE=67108864" "nopdl:BCL_PDL=0" "noll128:BCL_LL128=0"; do
  tag=${v%%:*}; envs=${v#*:}
  p=$((p+1))
  env $envs timeout 300 $TR --master-port $p bench.py --gpus 4 --no-sweep > $OUT/$tag.json 2> $OUT/$tag.err
  echo "$tag rc=$? $(tail -1 $OUT/$tag.json | python3 -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["e2e"]["value"], d["e2e"]["latency_ms"])' 2>&1 | tail -1)"
done
