cd "$(dirname "$0")/.."
mkdir -p gpurun_out/llchain
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/llchain/tests.log 2>&1; echo "rc=$?" >> gpurun_out/llchain/tests.log
for N in 4 2; do for P in ll pull; do
PROTO=$P SIZES=262144,1048576,2097152,4194304,8388608 CHUNKS=262144 ITERS=15 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 3030$N tools/sweep_opts.py >> gpurun_out/llchain/sweep_n$N.log 2>&1
done; done
