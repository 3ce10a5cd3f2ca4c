# Timings of library variants (tools/build_variant.sh): fused-kernel ms per config.
mkdir -p gpurun_out/var
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/var/smi.txt 2>&1
for v in ${VARIANTS}; do
  echo "== $v"
  RSOT_LIB_PATH=paper_2507_23602_b200/lib/var_$v.so timeout 600 python tools/trunc_timing.py ${CFGS:-cfg5 cfg3} 2>&1 | tail -4
done
