# timings + DRAM traffic of the fused truncated kernels (no tests)
for wl in cfg5 cfg3; do timeout 300 python tools/trunc_timing.py $wl; done
RSOT_PRECISION=fp32 timeout 300 python tools/trunc_timing.py cfg5 cfg3
for spec in "cfg5 fp64" "cfg3 fp64"; do
  set -- $spec
  RSOT_PRECISION=$2 timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum \
    --clock-control none -k regex:"^trunc_fused(32)?$" -s 1 -c 1 python tools/prof_trunc.py $1 2 2>&1 | grep -E "dram__|lts__|gpu__time" | sed "s/^/$1 $2 /"
done
