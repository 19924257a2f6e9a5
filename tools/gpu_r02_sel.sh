set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_index.py tests/test_gpu_guard.py tests/test_gpu_configs.py > gpurun_out/sel_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/sel_pytest.log
timeout 300 python bench.py --seq 4096 --hq 8 --hkv 1 --no-cpu-baseline --no-e2e --steps 20 --warmup 5 > gpurun_out/sel_c1_bench.json 2>&1; echo "c1 rc=$?"
timeout 300 python tools/live_kernel_times.py --seq 4096 --hq 8 --hkv 1 > gpurun_out/sel_c1_live.json 2> gpurun_out/sel_c1_live.err; echo "live rc=$?"
timeout 300 ncu --set full --import-source on -k regex:stage1_scores -c 1 -o gpurun_out/r02_c1_stage1 python tools/live_kernel_times.py --seq 4096 --hq 8 --hkv 1 --steps 1 --warmup 1 > gpurun_out/sel_ncu.log 2>&1; echo "ncu rc=$?"
