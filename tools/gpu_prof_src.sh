# --set full captures (with source) of the hot truncated kernels: cfg5 fp64, cfg5 fp32, cfg3 fp64
mkdir -p gpurun_out/src
for spec in "cfg5 fp64 trunc_fused" "cfg5 fp32 trunc_fused32" "cfg3 fp64 trunc_fused"; do
  set -- $spec
  RSOT_PRECISION=$2 timeout 600 python tools/prof_trunc.py $1 2 > gpurun_out/src/plain_$1_$2.log 2>&1; echo plain $1 $2 = $?
  RSOT_PRECISION=$2 timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"^$3$" -s 1 -c 1 \
    -o gpurun_out/src/full_$1_$2 -f python tools/prof_trunc.py $1 2 > gpurun_out/src/ncu_$1_$2.log 2>&1; echo full $1 $2 = $?
done
ls -la gpurun_out/src
