# Same box, two libraries: the sweep up to 1 MiB (single-call and 50 back-to-back calls) at N=2 and N=4.
OUT=gpurun_out/ab_lib
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
p=29700
for rep in 1; do
for lib in build/var_old/libbcl.so paper_1707_09414_b200/libbcl.so; do
  for n in 2 4; do
    p=$((p+1))
    tag=$(basename $(dirname $lib))_n${n}_r$rep
    BCL_LIB=$PWD/$lib CUDA_VISIBLE_DEVICES=0,1,2,3 timeout 600 $TR --nproc-per-node $n --master-port $p bench.py --gpus $n --sweep-max 1048576 --steps 5 --warmup 3 > $OUT/$tag.json 2>/dev/null
  done
done
done
