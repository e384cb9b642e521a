#!/bin/bash
# LL128 direct CTAs per rank (64 default vs 148 / 296), n = 4 and 2, single calls and 8 back to back.
out=gpurun_out/d128ctas; mkdir -p $out
(cd paper_1707_09414_b200 && make -s >/dev/null)
S=262144,524288,1048576,2097152
for n in 4 2; do
  devs=$( [ $n = 2 ] && echo 0,1 || echo 0,1,2,3 )
  for b2b in 8 1; do
    CUDA_VISIBLE_DEVICES=$devs SIZES=$S ITERS=15 B2B=$b2b ALGO=direct VARIANTS="auto;auto:ll128_direct_ctas=32;auto:ll128_direct_ctas=148;auto:ll128_direct_ctas=296" \
      timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2965$n \
      tools/r2/proto_ab.py 2>&1 | grep "N=" | tee -a $out/ab.txt
  done
done
