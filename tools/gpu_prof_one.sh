# One --set full capture of a truncated kernel: KREGEX, WL (workload), PREC.
mkdir -p gpurun_out
T="python tools/prof_trunc.py ${WL:-cfg5} 2"
RSOT_PRECISION=${PREC:-fp64} timeout 600 $T > gpurun_out/p1_plain.log 2>&1; echo plain=$?
RSOT_PRECISION=${PREC:-fp64} timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-trunc_fused}" -s 1 -c 1 \
  -o gpurun_out/${OUT:-one} -f $T > gpurun_out/p1_ncu.log 2>&1; echo full=$?
tail -2 gpurun_out/p1_ncu.log
