# Full GPU test suite + the cfg4 solve line (bench.py --workload cfg4).
mkdir -p gpurun_out/t2
timeout 1400 python -m pytest tests -m gpu -q > gpurun_out/t2/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/t2/pytest_gpu.log
timeout 900 python bench.py --workload cfg4 > gpurun_out/t2/cfg4.json 2> gpurun_out/t2/cfg4.err; echo cfg4_rc=$?
cat gpurun_out/t2/cfg4.json; tail -3 gpurun_out/t2/cfg4.err
