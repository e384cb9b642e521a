cd "$(dirname "$0")/.."
mkdir -p gpurun_out/ll128c
PROTO=ll128 SWEEP='BCL_LL128_CTAS=296;BCL_LL128_CTAS=444;BCL_LL128_CTAS=592' SIZES=4194304,16777216,67108864,134217728 CHUNKS=65536 ITERS=15 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 30701 tools/sweep_opts.py > gpurun_out/ll128c/n4.log 2>&1
