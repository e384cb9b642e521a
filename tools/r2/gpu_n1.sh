# 1-GPU pass: GPU tests, smoke, the N=1 bench, its ncu launch list and a full
# capture of the top kernel (after the plain run exited 0).
set -x
OUT=gpurun_out/r2_n1
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $OUT/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"; cat $OUT/bench.json
timeout 600 python bench.py --steps 3 --warmup 3 --cpu-iters 1 > $OUT/plain_small.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 3 --cpu-iters 1 > $OUT/ncu_launches.log 2>&1
echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:local_chain_kernel -s 4 -c 1 -o $OUT/prof_local_chain python bench.py --steps 3 --warmup 3 --cpu-iters 1 > $OUT/ncu_full.log 2>&1
echo "ncu full rc=$?"; tail -2 $OUT/ncu_full.log
