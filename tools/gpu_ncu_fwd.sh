set -x
timeout 600 python -m pytest tests/test_gpu_attn_fwd.py -q -x > gpurun_out/v11b_fwd_pytest.log 2>&1; echo "fwd tests rc=$?"
timeout 300 python tools/prof_step.py --seq 524288 --reps 1 > gpurun_out/ps2.log 2>&1; echo "plain rc=$?"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:attn_fwd_kernel -c 1 -o gpurun_out/r01v11_fwd python tools/prof_step.py --seq 524288 --reps 1 > gpurun_out/r01v11_ncu_fwd.log 2>&1; echo "ncu fwd rc=$?"
