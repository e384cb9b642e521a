cd "$(dirname "$0")/.."
mkdir -p gpurun_out/direct
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/direct/tests.log 2>&1; echo "rc=$?" >> gpurun_out/direct/tests.log
PROTO=pull SIZES=65536,1048576,8388608,67108864 CHUNKS=65536 ITERS=15 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 30901 tools/sweep_opts.py > gpurun_out/direct/n2.log 2>&1
PROTO=pull SIZES=65536,1048576,8388608,67108864 CHUNKS=65536 ITERS=10 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 30902 tools/sweep_opts.py > gpurun_out/direct/n4.log 2>&1
