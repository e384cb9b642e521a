cd "$(dirname "$0")/.."
rm -f gpurun_out/lc_var.log
for rep in 1 2; do for L in libbcl.so libbcl_lc_8_2.so libbcl_lc_16_2.so libbcl_lc_4_8.so libbcl_lc_8_5.so libbcl_lc_12_3.so; do
echo "== $L" >> gpurun_out/lc_var.log
BCL_LIB=$PWD/paper_1707_09414_b200/$L CHUNKS=524288 SWEEP="BCL_LOCAL_ITEM=16384;BCL_LOCAL_ITEM=4096" timeout 120 python tools/sweep_n1.py 2>&1 | grep "^\[" >> gpurun_out/lc_var.log
done; done
