cd "$(dirname "$0")/.."
for B in 4096 65536 1048576 4194304 8388608; do
echo "== $B" >> gpurun_out/n1_small.log
BYTES=$B CHUNKS=524288 SWEEP="BCL_LL_CHAIN_MAX=0" timeout 120 python tools/sweep_n1.py 2>&1 | grep "^\[" >> gpurun_out/n1_small.log
done
