# Last checks on the final tree (4 GPUs): the GPU suite on 4 GPUs and on GPU 0 alone, smoke(), the PCIe topology probe.
OUT=gpurun_out/r2final4; mkdir -p $OUT
(cd paper_1707_09414_b200 && make -s >/dev/null)
timeout 1200 python -m pytest tests -q -m gpu > $OUT/pytest_gpu_4gpu.log 2>&1
echo "pytest 4gpu rc=$? $(tail -1 $OUT/pytest_gpu_4gpu.log)"
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests -q -m gpu > $OUT/pytest_gpu_1gpu.log 2>&1
echo "pytest 1gpu rc=$? $(tail -1 $OUT/pytest_gpu_1gpu.log)"
CUDA_VISIBLE_DEVICES=0 timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_1gpu.log 2>&1
echo "smoke rc=$? $(tail -1 $OUT/smoke_1gpu.log)"
