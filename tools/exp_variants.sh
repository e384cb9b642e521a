#!/bin/bash
# Copy-path / occupancy experiment on >= 2 GPUs (single process, UVA).
cd "$(dirname "$0")/.."
D=${DEVICES:-0,1}
for sz in "67108864 524288" "1073741824 4194304" "1073741824 1048576"; do
  set -- $sz
  for v in ${VARIANTS:-"" "BCL_MAX_CTAS=296" "BCL_STAGES=2 BCL_STAGE_BYTES=8192" "BCL_STAGES=4 BCL_STAGE_BYTES=4096" "BCL_STAGES=3 BCL_STAGE_BYTES=8192" "BCL_SLICE_BYTES=65536" "BCL_SLICE_BYTES=65536 BCL_STAGES=4 BCL_STAGE_BYTES=4096"}; do
    env $v timeout 120 python tools/trace_chain.py --devices $D --bytes $1 --chunk $2 --quiet 2>&1 | tail -1
  done
done
