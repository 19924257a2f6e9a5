set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
timeout 900 python -m pytest -q -m gpu tests/test_gpu_xattn.py tests/test_gpu_index.py tests/test_gpu_guard.py > gpurun_out/xs3_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/xs3_pytest.log
timeout 600 python tools/live_kernel_times.py --seq 524288 --hq 16 --hkv 2 --xattn 0.9 --steps 2 --warmup 1 > gpurun_out/xs3_xattn_live.json 2> gpurun_out/xs3_xattn_live.err; echo "xlive rc=$?"; tail -3 gpurun_out/xs3_xattn_live.err
MT_XATTN_PAIR=0 timeout 600 python tools/live_kernel_times.py --seq 524288 --hq 16 --hkv 2 --xattn 0.9 --steps 2 --warmup 1 > gpurun_out/xs3_xattn_live_nopair.json 2> gpurun_out/xs3_xattn_live_nopair.err; echo "xlive0 rc=$?"
timeout 900 python tools/xattn_bench.py --tau 0.9 > gpurun_out/xs3_bench_tc.json 2> gpurun_out/xs3_bench_tc.err; echo "xb rc=$?"
timeout 300 python bench.py --seq 4096 --hq 8 --hkv 1 --no-cpu-baseline --no-e2e --steps 20 --warmup 5 > gpurun_out/xs3_c1.json 2>&1; echo "c1 rc=$?"
timeout 300 python tools/live_kernel_times.py --seq 4096 --hq 8 --hkv 1 > gpurun_out/xs3_c1_live.json 2> gpurun_out/xs3_c1_live.err; echo "live rc=$?"
