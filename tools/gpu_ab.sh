# A/B of library variants: parity tests on the default build, then timings per variant
mkdir -p gpurun_out/ab
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/ab/pytest_gpu.log
for v in ${VARIANTS}; do
  echo "== $v"
  RSOT_LIB_PATH=$v timeout 300 python bench.py --no-cpu-baseline --steps 10 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('cfg2', d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'])"
  RSOT_LIB_PATH=$v timeout 300 python tools/trunc_timing.py ${CFGS:-cfg5 cfg3}
  RSOT_PRECISION=fp32 RSOT_LIB_PATH=$v timeout 300 python tools/trunc_timing.py ${CFGS32:-}
done
