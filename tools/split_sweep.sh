python -m pytest tests -x -q -m gpu > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log; grep -E "^E " gpurun_out/t.log | head -8
for w in cfg3 cfg5; do echo "$w fp32"; RSOT_PRECISION=fp32 timeout 600 python tools/shard_diag.py $w 8 2>&1 | grep -E 'all|rank|Error'; done
for w in cfg3 cfg5; do python bench.py --workload $w --precision fp32 --steps 10 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"$w fp32\", d[\"ms_per_step\"])"; done
