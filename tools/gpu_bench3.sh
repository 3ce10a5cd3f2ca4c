# Bench lines: default (cfg5 fp64), cfg5 fp32, cfg3 fp64 and the reference arm (cfg5).
mkdir -p gpurun_out/b
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/b/cfg5.json 2> gpurun_out/b/cfg5.err; echo cfg5_rc=$?
timeout 900 python bench.py --steps 20 --warmup 5 --precision fp32 --no-cpu-baseline > gpurun_out/b/cfg5_fp32.json 2> gpurun_out/b/cfg5_fp32.err; echo fp32_rc=$?
timeout 900 python bench.py --steps 20 --warmup 5 --workload cfg3 --no-cpu-baseline > gpurun_out/b/cfg3.json 2> gpurun_out/b/cfg3.err; echo cfg3_rc=$?
timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/b/ref.json 2> gpurun_out/b/ref.err; echo ref_rc=$?
for f in cfg5 cfg5_fp32 cfg3 ref; do tail -c 1500 gpurun_out/b/$f.json; echo; done
