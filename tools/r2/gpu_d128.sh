#!/bin/bash
# LL128 direct: parity (new test, LL128 stress, soak with it on), then A/Bs at n = 4 and n = 2.
out=gpurun_out/d128; mkdir -p $out
timeout 600 python -m pytest tests/test_multigpu.py -x -q -k "ll128 or group or graph" 2>&1 | tail -5 | tee $out/pytest.txt
BCL_LL128_DIRECT_MIN=65536 timeout 400 python tools/r2/soak.py 600 5 2>&1 | tail -3 | tee $out/soak4.txt
tools/r2/ab_d128.sh 4
CUDA_VISIBLE_DEVICES=0,1 tools/r2/ab_d128.sh 2
