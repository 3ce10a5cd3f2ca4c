mkdir -p gpurun_out
timeout 600 python tools/prof_trunc.py cfg5 2 > gpurun_out/plain_t.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:trunc_fused -s 1 -c 1 -o gpurun_out/prof_cfg5 python tools/prof_trunc.py cfg5 2 > gpurun_out/ncu_t.log 2>&1; echo rc=$?
tail -3 gpurun_out/ncu_t.log
