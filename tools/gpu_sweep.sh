mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/pytest_gpu.log | grep -v "^$"
for c in ${CPRS:-3}; do RSOT_CELLS_PER_RADIUS=$c timeout 600 python tools/trunc_timing.py cfg3 cfg5; done
