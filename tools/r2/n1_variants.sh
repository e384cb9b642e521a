# N=1 config 1 under build variants (unroll x min blocks) and item sizes.
for v in build/var_*; do
  BCL_LIB=$v/libbcl.so SWEEP="${SWEEP:-BCL_LOCAL_ITEM=4096;BCL_LOCAL_ITEM=8192;BCL_LOCAL_CLAIM=0}" timeout 300 python tools/sweep_n1.py 2>&1 | sed "s|^|$(basename $v) |" | grep "\["
done
