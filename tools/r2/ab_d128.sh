#!/bin/bash
# LL128 direct vs 16-byte LL direct (and the tuned choice) at n = $1, single
# calls and 8 back to back; sizes 16 KiB - 2 MiB.
n=${1:-2}
out=gpurun_out/d128; mkdir -p $out
S=16384,65536,131072,262144,524288,1048576,2097152
for b2b in 1 8; do
  for algo in direct table; do
    SIZES=$S ITERS=15 B2B=$b2b ALGO=$algo VARIANTS="auto;auto:ll128_direct_min=65536;auto:ll128_direct_min=16384" \
      timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29611 \
      tools/r2/proto_ab.py 2>&1 | grep -v Warning | grep "N=" | tee -a $out/ab_n$n.txt
  done
done
