cd "$(dirname "$0")/.."
mkdir -p gpurun_out/mbox
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/mbox/tests.log 2>&1; echo "rc=$?" >> gpurun_out/mbox/tests.log
PROTO=pull SIZES=65536,1048576,8388608,67108864 CHUNKS=65536 ITERS=15 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 30901 tools/sweep_opts.py > gpurun_out/mbox/n2.log 2>&1
PROTO=pull SIZES=65536,1048576,8388608,67108864,268435456 CHUNKS=65536 ITERS=10 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 30902 tools/sweep_opts.py > gpurun_out/mbox/n4.log 2>&1
TRACE_ITERS=10 TRACE_BYTES=67108864 TRACE_CHUNK=65536 TRACE_NPZ=gpurun_out/mbox/n2trace_rRANK.npz timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 30903 tools/trace_mp.py 2>&1 | grep "^rank" > gpurun_out/mbox/n2trace.log
