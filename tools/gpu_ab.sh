timeout 600 python -m pytest tests/test_gpu_attn_fwd.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -1
timeout 300 python tools/fwd_step_timeline.py 4 1 2 2>&1 | grep "step time" | tail -1
timeout 300 python tools/fwd_step_timeline.py 4 1 0 2>&1 | grep "step time" | tail -1
