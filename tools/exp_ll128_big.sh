cd "$(dirname "$0")/.."
mkdir -p gpurun_out/ll128big
for N in 4 2; do for P in ll128 pull; do
BCL_LL128_MAX=268435456 PROTO=$P SIZES=33554432,67108864,134217728,268435456 CHUNKS=65536 ITERS=10 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 3050$N tools/sweep_opts.py >> gpurun_out/ll128big/sweep_n$N.log 2>&1
done; done
