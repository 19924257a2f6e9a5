timeout 600 python -m pytest tests/test_gpu_attn_bwd.py tests/test_gpu_attn_fwd.py -x -q 2>&1 | tail -1
timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['phase_ms'])"
