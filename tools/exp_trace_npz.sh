mkdir -p gpurun_out/npz
for c in 65536 524288; do
TRACE_ITERS=10 TRACE_BYTES=67108864 TRACE_CHUNK=$c TRACE_NPZ=gpurun_out/npz/n4_c${c}_rRANK.npz timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 30141 tools/trace_mp.py 2>&1 | grep "^rank [0-9]:" >> gpurun_out/npz/log
done
