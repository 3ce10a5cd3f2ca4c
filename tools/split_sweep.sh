python -m pytest tests -x -q -m gpu > gpurun_out/t.log 2>&1; tail -2 gpurun_out/t.log; grep -E "^E " gpurun_out/t.log | head -8
timeout 600 python tools/shard_diag.py cfg3 8 2>&1 | grep -E "all|rank|Error"
python bench.py --workload cfg3 --steps 10 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"cfg3 default\", d[\"ms_per_step\"], d[\"gpu_launches\"])"
