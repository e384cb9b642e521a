set -x
N=$(nvidia-smi -L | wc -l)
OUT=gpurun_out/r2ab2_n$N
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
VARIANTS="pull;pull:writer_fence=2;pull:strict_sys=1;pull:stage_bytes=4096;pull:max_ctas=74;pull:window_bytes=2097152;pull:window_bytes=1048576;pull:stage_bytes=4096,window_bytes=2097152;pull:stages=3,stage_bytes=4096;push;push:window_bytes=2097152" SIZES=8388608,67108864,268435456,1073741824 timeout 1500 $TR --master-port 29530 tools/r2/proto_ab.py > $OUT/proto_ab.log 2>&1; echo "ab rc=$?"; grep "^N=" $OUT/proto_ab.log
