python tools/cfg4_prepare.py /tmp/cfg4s small > /dev/null
RSOT_DUMP_PSI=gpurun_out/cfg4s_gpu_psi.f64 timeout 300 ./paper_2507_23602_b200/lib/cfg4_solve /tmp/cfg4s 1e-8 1000 > gpurun_out/cfg4s_gpu.json 2>&1; echo rc=$?
cat gpurun_out/cfg4s_gpu.json
