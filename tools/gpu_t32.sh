RSOT_PRECISION=fp32 timeout 300 python tools/trunc_timing.py cfg5 cfg3
timeout 900 python -m pytest tests/test_gpu_fp32.py -x -q 2>&1 | tail -2
