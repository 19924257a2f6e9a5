MT_BWD_DBG=4 timeout 600 python -m pytest tests/test_gpu_attn_bwd.py -x -q 2>&1 | tail -1
for dbg in 0 4 1; do MT_BWD_DBG=$dbg timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('dbg=$dbg', d['value'], d['roofline']['phase_ms'])"; done
