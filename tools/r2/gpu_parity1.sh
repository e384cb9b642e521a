set -x
nvidia-smi -L
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2_pytest1.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1
echo smoke rc=$?
tail -3 gpurun_out/r2_pytest1.log; tail -3 gpurun_out/r2_smoke.log
