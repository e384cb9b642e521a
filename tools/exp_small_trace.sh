mkdir -p gpurun_out/small
for n in 2 4; do for m in 65536 1048576; do
 echo "== n=$n m=$m" >> gpurun_out/small/log
 TRACE_BYTES=$m TRACE_CHUNK=65536 timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 3011$n tools/trace_mp.py >> gpurun_out/small/log 2>&1
done; done
