mkdir -p gpurun_out/ev
python bench.py > gpurun_out/ev/bench_cfg2.json 2> gpurun_out/ev/bench_cfg2.err; echo bench_cfg2=$?
python bench.py --workload cfg5 > gpurun_out/ev/bench_cfg5.json 2> gpurun_out/ev/bench_cfg5.err; echo bench_cfg5=$?
python bench.py --workload cfg5 --precision fp32 --no-cpu-baseline > gpurun_out/ev/bench_cfg5_fp32.json 2>&1; echo bench_cfg5_fp32=$?
python bench.py --workload cfg3 --no-cpu-baseline > gpurun_out/ev/bench_cfg3.json 2>&1; echo bench_cfg3=$?
python bench.py --workload cfg3 --precision fp32 --no-cpu-baseline > gpurun_out/ev/bench_cfg3_fp32.json 2>&1; echo bench_cfg3_fp32=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev/bench_ref_cfg2.json 2>&1; echo ref=$?
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev/launches_cfg2.csv $B > /dev/null 2>&1; echo l2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_pass -s 2 -c 2 -o gpurun_out/ev/full_cfg2 -f $B > /dev/null 2>&1; echo f2=$?
