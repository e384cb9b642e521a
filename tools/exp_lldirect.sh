cd "$(dirname "$0")/.."
mkdir -p gpurun_out/lld
rm -f gpurun_out/lld/ab3.log
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/lld/tests.log 2>&1; echo "rc=$?" >> gpurun_out/lld/tests.log
for rep in 1 2 3; do for L in libbcl.so libbcl_old.so; do
echo "== $L" >> gpurun_out/lld/ab3.log
BCL_LIB=$PWD/paper_1707_09414_b200/$L ALGO=direct SIZES=4,65536,524288 CHUNKS=0 ITERS=60 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 3060$rep tools/sweep_opts.py 2>&1 | grep "^\[" >> gpurun_out/lld/ab3.log
done; done
