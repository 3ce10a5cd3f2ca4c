mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 $B > gpurun_out/plain_d.log 2>&1; echo plain=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_pass -s 2 -c 2 -o gpurun_out/${OUT:-prof_cfg2} -f $B > gpurun_out/ncu_d.log 2>&1; echo rc=$?
