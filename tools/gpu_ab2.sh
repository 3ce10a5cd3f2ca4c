# A/B of library variants on the GPU box: quick parity tests on the default
# build, then fused-kernel timings (tools/trunc_timing.py) per variant.
# usage (under gpurun): VARIANTS="base lean1" [TESTS="..."] bash tools/gpu_ab2.sh
mkdir -p gpurun_out/ab
timeout 900 python -m pytest ${TESTS:-tests/test_gpu_parity.py tests/test_gpu_fullsize.py} -m gpu -x -q > gpurun_out/ab/pytest.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/ab/pytest.log
for v in ${VARIANTS} default; do
  L=paper_2507_23602_b200/lib/var_$v.so; [ $v = default ] && L=paper_2507_23602_b200/lib/librsot_b200.so
  echo "== $v"
  RSOT_LIB_PATH=$L timeout 300 python tools/trunc_timing.py ${CFGS:-cfg5 cfg3} 2>&1 | tail -2
  if [ -n "$CFGS32" ]; then RSOT_PRECISION=fp32 RSOT_LIB_PATH=$L timeout 300 python tools/trunc_timing.py $CFGS32 2>&1 | tail -2; fi
done
