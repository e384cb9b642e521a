#!/bin/bash
# Re-tune the n = 2 / n = 4 tables below 4 MiB with LL128 direct on (default),
# raw latencies kept; spliced into the builtin table by hand (rows < 2965821).
out=gpurun_out/retune_small; mkdir -p $out
(cd paper_1707_09414_b200 && make -s >/dev/null)
for n in 4 2; do
  devs=$( [ $n = 2 ] && echo 0,1 || echo 0,1,2,3 )
  CUDA_VISIBLE_DEVICES=$devs timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2962$n tools/tune_b200.py --max-bytes 4194304 --iters 8 --cands direct,knomial,scatter_ring_allgather,chain_pipelined \
    --out $out/small_n$n.csv --raw $out/raw_small_n$n.csv > $out/tune_n$n.log 2>&1
  tail -25 $out/tune_n$n.log
done
