cd "$(dirname "$0")/.."
mkdir -p gpurun_out/quick
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/quick/n1.json 2>gpurun_out/quick/n1.err
BCL_WRITER_FENCE=0 timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/quick/n1_wf0.json 2>>gpurun_out/quick/n1.err
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/quick/n1b.json 2>>gpurun_out/quick/n1.err
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2990$N bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/quick/n$N.json 2> gpurun_out/quick/n$N.err
done
