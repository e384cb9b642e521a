#!/bin/bash
# Same-box A/B of the tuned choice, 50 calls back to back (the bench's b2b shape), n = 4 then 2:
# LL128 direct default (one CTA per SM) vs 64 CTAs vs 16-byte LL direct lines.
out=gpurun_out/d128b50; mkdir -p $out
(cd paper_1707_09414_b200 && make -s >/dev/null)
S=131072,262144,524288,1048576,2097152
for n in 4 2; do
  devs=$( [ $n = 2 ] && echo 0,1 || echo 0,1,2,3 )
  for rep in 1 2; do
    CUDA_VISIBLE_DEVICES=$devs SIZES=$S ITERS=10 B2B=50 ALGO=table VARIANTS="auto;auto:ll128_direct_ctas=64;auto:ll128_direct_min=0" \
      timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2966$n \
      tools/r2/proto_ab.py 2>&1 | grep "N=" | tee -a $out/ab.txt
  done
done
