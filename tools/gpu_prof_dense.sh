mkdir -p gpurun_out
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_d.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_pass -s 2 -c 2 -o gpurun_out/prof_cfg2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_d.log 2>&1; echo rc=$?
