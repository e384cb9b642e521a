#!/bin/bash
# multi-process trace across variants (N GPUs)
cd "$(dirname "$0")/.."
N=${N:-4}
P=29600
for v in "${@}"; do
  for sz in 67108864 1073741824; do
    P=$((P+1))
    echo "== $v bytes=$sz"
    env $v TRACE_BYTES=$sz timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $P tools/trace_mp.py 2>&1 | grep "^rank"
  done
done
