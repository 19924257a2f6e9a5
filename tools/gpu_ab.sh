timeout 600 python -m pytest tests/test_gpu_attn_bwd.py -x -q 2>&1 | tail -1
timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['phase_ms'])"
timeout 300 python tools/prof_step.py --seq 524288 --reps 1 > gpurun_out/ps.log 2>&1
timeout 1200 ncu --set full --clock-control none -k regex:attn_bwd_kernel --launch-skip 1 -c 1 -o gpurun_out/r01v4_bwd_bar2 python tools/prof_step.py --seq 524288 --reps 1 > gpurun_out/r01v4_ncu_bwd_bar2.log 2>&1; echo rc=$?
