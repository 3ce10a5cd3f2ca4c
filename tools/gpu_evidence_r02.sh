# Round-2 evidence: GPU tests, smoke, bench lines, reference arm,
# ncu launch lists and --set full captures of the hot kernels, cfg4 solve.
set -u
E=gpurun_out/ev; mkdir -p $E
timeout 1200 python -m pytest tests -m gpu -q > $E/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 $E/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $E/smoke.log 2>&1; echo smoke=$?
timeout 900 python bench.py --steps 20 --warmup 5 > $E/bench_cfg5.json 2> $E/bench_cfg5.err; echo bench_cfg5=$?
timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 > $E/bench_ref_cfg5.json 2> $E/bench_ref_cfg5.err; echo ref_cfg5=$?
timeout 900 python bench.py --workload cfg2 > $E/bench_cfg2.json 2> $E/bench_cfg2.err; echo bench_cfg2=$?
timeout 900 python bench.py --workload cfg2 --impl reference --steps 3 --warmup 1 > $E/bench_ref_cfg2.json 2>&1; echo ref_cfg2=$?
timeout 900 python bench.py --workload cfg4 > $E/bench_cfg4.json 2> $E/bench_cfg4.err; echo bench_cfg4=$?
for wl in cfg5 cfg3; do for p in fp64 fp32; do
  timeout 900 python bench.py --workload $wl --precision $p --no-cpu-baseline > $E/bench_${wl}_$p.json 2> $E/bench_${wl}_$p.err; echo bench_${wl}_$p=$?
done; done
B="python bench.py --workload cfg2 --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $E/launches_cfg2.csv $B > /dev/null 2>&1; echo l_cfg2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_pass -s 2 -c 2 -o $E/full_cfg2 -f $B > /dev/null 2>&1; echo f_cfg2=$?
for spec in "cfg5 fp64" "cfg3 fp64" "cfg5 fp32"; do
  set -- $spec; W=$1; P=$2
  T="python tools/prof_trunc.py $W 2"
  RSOT_PRECISION=$P timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $E/launches_${W}_$P.csv $T > /dev/null 2>&1; echo l_${W}_$P=$?
  RSOT_PRECISION=$P timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"^trunc_fused(32)?$|trunc_nearest" -s 2 -c 2 -o $E/full_${W}_$P -f $T > /dev/null 2>&1; echo f_${W}_$P=$?
done
ls -la $E
# summaries on the box (the raw reports exceed gpurun's 64 MiB return limit)
N="round 2, commit $(cat .commit 2>/dev/null || echo HEAD)"
python tools/ncu_summary.py --rep $E/full_cfg2.ncu-rep --launches $E/launches_cfg2.csv --out $E/r02_cfg2 \
  --note "$N: cfg2 dense (bench.py --steps 2 --warmup 3); --set full = one evaluation's pass A + pass B" \
  --traffic-out $E/ncu_summary_cfg2.json > /dev/null; echo s_cfg2=$?
for spec in "cfg5 fp64" "cfg3 fp64" "cfg5 fp32"; do
  set -- $spec; W=$1; P=$2; suf=""; [ $P = fp32 ] && suf="_fp32"
  python tools/ncu_summary.py --rep $E/full_${W}_$P.ncu-rep --launches $E/launches_${W}_$P.csv --out $E/r02_${W}_$P \
    --note "$N: $W $P (tools/prof_trunc.py $W 2); --set full = the second evaluation's fused kernel + nearest kernel" \
    --traffic-out $E/ncu_summary_${W}${suf}.json > /dev/null; echo s_${W}_$P=$?
  ncu -i $E/full_${W}_$P.ncu-rep --page source --csv --print-source sass > $E/sass_${W}_$P.csv 2>/dev/null
  python tools/ncu_sass_hot.py $E/sass_${W}_$P.csv > $E/r02_${W}_${P}_hot.txt 2>&1; echo h_${W}_$P=$?
  python tools/ncu_src_lines.py $E/full_${W}_$P.ncu-rep 60 > $E/r02_${W}_${P}_lines.txt 2>&1
  rm -f $E/sass_${W}_$P.csv
done
ncu -i $E/full_cfg2.ncu-rep --page source --csv --print-source sass > $E/sass_cfg2.csv 2>/dev/null
python tools/ncu_sass_hot.py $E/sass_cfg2.csv > $E/r02_cfg2_hot.txt 2>&1; rm -f $E/sass_cfg2.csv
mkdir -p gpurun_out/rep; mv $E/full_cfg2.ncu-rep gpurun_out/rep/; rm -f $E/*.ncu-rep
du -sh gpurun_out
rm -f $E/full_*.ncu-rep
ls -la $E
