# Round-2 GPU check: full GPU test suite (incl. full-size parity vs the
# reference fixtures), the default bench (cfg5 fp64) and the reference arm.
mkdir -p gpurun_out/r02
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/r02/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r02/pytest_gpu.log
if [ -z "${SKIP_BENCH:-}" ]; then
  timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02/bench.json 2> gpurun_out/r02/bench.err; echo bench_rc=$?
  tail -c 3000 gpurun_out/r02/bench.json
  timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02/ref.json 2> gpurun_out/r02/ref.err; echo ref_rc=$?
  tail -c 2000 gpurun_out/r02/ref.json
fi
