mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dropin.py -x -q 2>&1 | tail -3
python tools/cfg4_prepare.py /tmp/cfg4 > /dev/null
timeout ${CFG4_TIMEOUT:-1200} ./paper_2507_23602_b200/lib/cfg4_solve /tmp/cfg4 ${CFG4_TOL:-1e-8} ${CFG4_MAXIT:-1000} > gpurun_out/cfg4.json 2> gpurun_out/cfg4.err; echo cfg4_rc=$?
cat gpurun_out/cfg4.json; tail -3 gpurun_out/cfg4.err
