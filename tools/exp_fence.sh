#!/bin/bash
cd "$(dirname "$0")/.."
D=${DEVICES:-0,1,2,3}
V=(
"BCL_WINDOW_BYTES=16777216 BCL_MIN_SLICE=16384"
"BCL_WINDOW_BYTES=16777216 BCL_MIN_SLICE=16384 BCL_FENCE=1"
"BCL_WINDOW_BYTES=16777216 BCL_MIN_SLICE=16384 BCL_FENCE=2"
"BCL_WINDOW_BYTES=4194304 BCL_MIN_SLICE=2048 BCL_FENCE=2"
"BCL_WINDOW_BYTES=4194304 BCL_MIN_SLICE=2048 BCL_PUB_EVERY=4"
"BCL_WINDOW_BYTES=4194304 BCL_MIN_SLICE=8192"
"BCL_WINDOW_BYTES=4194304 BCL_MIN_SLICE=8192 BCL_FENCE=2"
"BCL_WINDOW_BYTES=4194304 BCL_MIN_SLICE=8192 BCL_FENCE=1"
)
for v in "${V[@]}"; do
  for sz in "67108864 524288" "1073741824 4194304"; do
    set -- $sz
    env $v timeout 60 python tools/trace_chain.py --devices $D --bytes $1 --chunk $2 --quiet 2>&1 | tail -1
  done
done
for v in "${V[0]}" "${V[3]}" "${V[5]}"; do
  env $v timeout 60 python tools/trace_chain.py --devices $D 2>&1 | grep -v "^rank 0"
done
