cd "$(dirname "$0")/.."
mkdir -p gpurun_out/final
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/final/tests.log 2>&1; echo "rc=$?" >> gpurun_out/final/tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/final/smoke.log
for P in ll128 pull; do
BCL_LL128_MAX=536870912 PROTO=$P SIZES=134217728,268435456,536870912 CHUNKS=131072 ITERS=6 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 3110$([ $P = pull ] && echo 1 || echo 2) tools/sweep_opts.py >> gpurun_out/final/ll128_big.log 2>&1
done
