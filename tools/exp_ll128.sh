cd "$(dirname "$0")/.."
mkdir -p gpurun_out/ll128
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/ll128/tests_all.log 2>&1; echo "rc=$?" >> gpurun_out/ll128/tests_all.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29904 bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/ll128/bench_n4.json 2> gpurun_out/ll128/bench_n4.err
