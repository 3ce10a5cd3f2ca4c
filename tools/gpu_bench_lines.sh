# bench lines only (kernels unchanged since the last ncu evidence)
E=gpurun_out/bl; mkdir -p $E
timeout 900 python bench.py > $E/bench_cfg2.json 2> $E/bench_cfg2.err; echo bench_cfg2=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $E/bench_ref_cfg2.json 2>&1; echo ref_cfg2=$?
for wl in cfg5 cfg3; do for p in fp64 fp32; do
  timeout 900 python bench.py --workload $wl --precision $p --no-cpu-baseline > $E/bench_${wl}_$p.json 2> $E/bench_${wl}_$p.err; echo bench_${wl}_$p=$?
done; done
timeout 900 python bench.py --workload cfg5 --steps 3 > $E/bench_cfg5_cpu.json 2> $E/bench_cfg5_cpu.err; echo bench_cfg5_cpu=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $E/smoke.log 2>&1; echo smoke=$?
