# cfg4 full solve on the GPU drop-in with the potentials entering every stage
# dumped (for the CPU reference's per-stage runs), then one --set full ncu
# capture (with source) of the cfg5 fp64 fused kernel.
mkdir -p gpurun_out/c4 gpurun_out/src
python tools/cfg4_prepare.py /tmp/cfg4 > gpurun_out/c4/prepare.log 2>&1
RSOT_DUMP_STAGE_PSI=gpurun_out/c4/psi timeout 900 paper_2507_23602_b200/lib/cfg4_solve /tmp/cfg4 1e-8 > gpurun_out/c4/cfg4_solve_gpu.json 2> gpurun_out/c4/cfg4_solve_gpu.err; echo cfg4_rc=$?
cat gpurun_out/c4/cfg4_solve_gpu.json
timeout 600 python tools/prof_trunc.py cfg5 2 > gpurun_out/src/plain_cfg5.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"^trunc_fused$" -s 1 -c 1 \
  -o gpurun_out/src/r02_cfg5_fp64 -f python tools/prof_trunc.py cfg5 2 > gpurun_out/src/ncu_cfg5.log 2>&1; echo ncu_rc=$?
ls -la gpurun_out/src
