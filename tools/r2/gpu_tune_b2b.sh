#!/bin/bash
# Tables from the back-to-back oracle (mean of 8 calls issued back to back) up to 16 MiB, n = 4 and n = 2.
out=gpurun_out/tune_b2b; mkdir -p $out
(cd paper_1707_09414_b200 && make -s >/dev/null)
for n in 4 2; do
  devs=$( [ $n = 2 ] && echo 0,1 || echo 0,1,2,3 )
  CUDA_VISIBLE_DEVICES=$devs timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2964$n tools/tune_b200.py --max-bytes 16777216 --iters 6 --b2b 8 \
    --out $out/b2b_n$n.csv --raw $out/raw_b2b_n$n.csv > $out/tune_n$n.log 2>&1
  tail -22 $out/tune_n$n.log
done
