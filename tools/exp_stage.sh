#!/bin/bash
cd "$(dirname "$0")/.."
D=${DEVICES:-0,1,2,3}
for v in ${VARIANTS:-"BCL_STAGE_BYTES=0" "BCL_STAGE_BYTES=4096" "BCL_STAGE_BYTES=8192" "BCL_STAGE_BYTES=8192 BCL_WINDOW_BYTES=8388608" "BCL_STAGE_BYTES=12288 BCL_MIN_SLICE=8192"}; do
  for sz in "67108864 524288" "1073741824 4194304" "1073741824 1048576"; do
    set -- $sz
    env $v timeout 60 python tools/trace_chain.py --devices $D --bytes $1 --chunk $2 --quiet 2>&1 | tail -1
  done
done
