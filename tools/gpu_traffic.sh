# parity tests + timings + DRAM traffic / L2 hit rate of the fused truncated kernels
VARIANTS=paper_2507_23602_b200/lib/librsot_b200.so CFGS32=cfg5 bash tools/gpu_ab.sh
for spec in "cfg5 fp64" "cfg5 fp32" "cfg3 fp64"; do
  set -- $spec
  RSOT_PRECISION=$2 timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum \
    --clock-control none -k regex:"^trunc_fused(32)?$" -s 1 -c 1 python tools/prof_trunc.py $1 2 2>&1 | grep -E "dram__|lts__|gpu__time" | sed "s/^/$1 $2 /"
done
