# Same box: programmatic dependent launch on/off (BCL_PDL) -- sweep to 1 MiB at N=2/N=4 and ResNet-50 per tensor.
OUT=gpurun_out/ab_pdl
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
p=29800
for pdl in 0 1; do
  for n in 2 4; do
    p=$((p+1))
    BCL_PDL=$pdl CUDA_VISIBLE_DEVICES=0,1,2,3 timeout 150 $TR --nproc-per-node $n --master-port $p bench.py --gpus $n --sweep-max 1048576 --steps 5 --warmup 3 > $OUT/sweep_pdl${pdl}_n$n.json 2>/dev/null
  done
  for f in "" "--graph"; do
    p=$((p+1))
    BCL_PDL=$pdl timeout 150 $TR --nproc-per-node 4 --master-port $p bench.py --gpus 4 --workload resnet50 $f --steps 10 --warmup 3 > $OUT/resnet50_pdl${pdl}$(echo $f | tr -d ' -').json 2>/dev/null
  done
done
