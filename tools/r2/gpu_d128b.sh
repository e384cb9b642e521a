#!/bin/bash
# LL128 direct on by default (128 KiB): multi-GPU suites, soak, and the tuned choice vs LL direct (ll128_direct_min=0).
out=gpurun_out/d128b; mkdir -p $out
(cd paper_1707_09414_b200 && make -s >/dev/null)
timeout 700 python -m pytest tests/test_multigpu.py tests/test_nvls.py -x -q 2>&1 | tail -3 | tee $out/pytest4.txt
timeout 400 python tools/r2/soak.py 800 9 2>&1 | tail -3 | tee $out/soak4.txt
S=65536,131072,262144,524288,1048576,2097152,4194304
for n in 4 2; do
  devs=$( [ $n = 2 ] && echo 0,1 || echo 0,1,2,3 )
  for b2b in 1 8; do
    CUDA_VISIBLE_DEVICES=$devs SIZES=$S ITERS=15 B2B=$b2b ALGO=table VARIANTS="auto;auto:ll128_direct_min=0" \
      timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n \
      tools/r2/proto_ab.py 2>&1 | grep "N=" | tee -a $out/ab_table.txt
  done
done
