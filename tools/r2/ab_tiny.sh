#!/bin/bash
# Small messages at n = 2 / 4: `direct` (16-byte LL lines) vs the pipelined chain (LL128 lines), PDL on/off,
# single calls (40 samples) and 16 back to back.
out=gpurun_out/tiny; mkdir -p $out
(cd paper_1707_09414_b200 && make -s >/dev/null)
S=8,1024,4096,16384,65536,262144
for n in 2 4; do
  devs=$( [ $n = 2 ] && echo 0,1 || echo 0,1,2,3 )
  for pdl in 1 0; do
    for b2b in 1 16; do
      for algo in direct chain_pipelined; do
        BCL_PDL=$pdl CUDA_VISIBLE_DEVICES=$devs SIZES=$S ITERS=40 B2B=$b2b ALGO=$algo CHUNK=65536 VARIANTS="auto" \
          timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2963$n \
          tools/r2/proto_ab.py 2>&1 | grep "N=" | sed "s/^/pdl=$pdl /" | tee -a $out/ab_tiny.txt
      done
    done
  done
done
