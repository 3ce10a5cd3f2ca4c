# quick GPU check: parity tests + probe timings + cfg2 bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python tools/parity_probe.py > gpurun_out/probe.log 2>&1; echo probe_rc=$?
grep -E "FAIL|eval|ALLOK" gpurun_out/probe.log | grep -v "eval [12]:" 
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_cfg2.json 2>&1; echo bench_rc=$?
cat gpurun_out/bench_cfg2.json
