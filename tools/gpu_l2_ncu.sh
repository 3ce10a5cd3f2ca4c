# DRAM bytes of the fp64 fused kernel (cfg5, second evaluation): mask pool
# layout/L2 window A/B.
mkdir -p gpurun_out/l2
for v in old new; do
  RSOT_LIB_PATH=paper_2507_23602_b200/lib/var_$v.so timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum \
    --clock-control none -k regex:"^trunc_fused$" -s 1 -c 1 --csv python tools/prof_trunc.py cfg5 2 > gpurun_out/l2/ncu_$v.csv 2>&1; echo $v=$?
  grep -E "dram__bytes|hit_rate|duration" gpurun_out/l2/ncu_$v.csv | cut -c1-250
done
