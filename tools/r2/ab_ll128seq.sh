# Same box: LL128 with per-call ring reuse (var_old) vs ring positions continued across calls.
OUT=gpurun_out/ab_ll128seq
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
p=29900
for lib in build/var_old/libbcl.so paper_1707_09414_b200/libbcl.so; do
  tag=$(basename $(dirname $lib))
  for n in 2 4; do
    p=$((p+1))
    BCL_LIB=$PWD/$lib timeout 200 $TR --nproc-per-node $n --master-port $p bench.py --gpus $n --sweep-max 67108864 --b2b-max 16777216 --steps 5 --warmup 3 > $OUT/${tag}_n$n.json 2>/dev/null
  done
  p=$((p+1))
  BCL_LIB=$PWD/$lib timeout 150 $TR --nproc-per-node 4 --master-port $p bench.py --gpus 4 --workload resnet50 --steps 10 --warmup 3 > $OUT/${tag}_resnet50.json 2>/dev/null
done
