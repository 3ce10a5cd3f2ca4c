# full GPU check of HEAD: parity tests, smoke, bench lines per workload
mkdir -p gpurun_out/chk
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/chk/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/chk/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/chk/smoke.log 2>&1; echo smoke_rc=$?
timeout 600 python bench.py > gpurun_out/chk/bench_cfg2.json 2> gpurun_out/chk/bench_cfg2.err; echo bench_cfg2=$?
timeout 900 python bench.py --workload cfg5 --no-cpu-baseline > gpurun_out/chk/bench_cfg5.json 2>&1; echo bench_cfg5=$?
timeout 900 python bench.py --workload cfg5 --precision fp32 --no-cpu-baseline > gpurun_out/chk/bench_cfg5_fp32.json 2>&1; echo bench_cfg5_fp32=$?
timeout 900 python bench.py --workload cfg3 --no-cpu-baseline > gpurun_out/chk/bench_cfg3.json 2>&1; echo bench_cfg3=$?
timeout 900 python bench.py --workload cfg3 --precision fp32 --no-cpu-baseline > gpurun_out/chk/bench_cfg3_fp32.json 2>&1; echo bench_cfg3_fp32=$?
for f in gpurun_out/chk/bench_*.json; do echo $f; tail -c 600 $f; echo; done
