# Round profile capture: plain runs first (each ncu command only after the
# same command exited 0 without ncu), launch lists, one --set full capture
# of the top kernels.  Outputs in gpurun_out/; summarised by
# tools/ncu_summary.py into profiles/.
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 $B > gpurun_out/p_plain_cfg2.log 2>&1; echo plain_cfg2=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_cfg2.csv $B > gpurun_out/p_ncu1_cfg2.log 2>&1; echo launches_cfg2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_pass -s 2 -c 2 \
  -o gpurun_out/full_cfg2 -f $B > gpurun_out/p_ncu2_cfg2.log 2>&1; echo full_cfg2=$?
for W in cfg5 cfg3; do
  T="python tools/prof_trunc.py $W 2"
  timeout 600 $T > gpurun_out/p_plain_$W.log 2>&1; echo plain_$W=$?
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$W.csv $T > gpurun_out/p_ncu1_$W.log 2>&1; echo launches_$W=$?
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"trunc_fused|trunc_nearest" -s 2 -c 2 \
    -o gpurun_out/full_$W -f $T > gpurun_out/p_ncu2_$W.log 2>&1; echo full_$W=$?
done
ls -la gpurun_out | tail -20
