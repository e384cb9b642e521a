set -x
N=$(nvidia-smi -L | wc -l)
OUT=gpurun_out/r2ab_n$N
mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 900 $TR --master-port 29530 tools/r2/proto_ab.py > $OUT/proto_ab.log 2>&1; echo "ab rc=$?"; grep "^N=" $OUT/proto_ab.log
timeout 600 python -m pytest tests/test_transport_shim.py tests/test_multigpu.py -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.log
