# usage: W=cfg5 P=fp64 bash tools/gpu_evidence_trunc.sh
mkdir -p gpurun_out/ev
T="python tools/prof_trunc.py $W 2"
RSOT_PRECISION=$P timeout 600 $T > /dev/null 2>&1; echo plain_${W}_$P=$?
RSOT_PRECISION=$P timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev/launches_${W}_$P.csv $T > /dev/null 2>&1; echo l_${W}_$P=$?
RSOT_PRECISION=$P timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"trunc_fused|trunc_nearest" -s 2 -c 2 -o gpurun_out/ev/full_${W}_$P -f $T > /dev/null 2>&1; echo f_${W}_$P=$?
