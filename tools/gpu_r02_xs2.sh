set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
timeout 900 python -m pytest -q -m gpu tests/test_gpu_xattn.py tests/test_gpu_block_sparse.py > gpurun_out/xs2_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/xs2_pytest.log
timeout 600 python tools/live_kernel_times.py --seq 524288 --hq 16 --hkv 2 --xattn 0.9 --steps 2 --warmup 1 > gpurun_out/xs2_xattn_live.json 2> gpurun_out/xs2_xattn_live.err; echo "xlive rc=$?"; tail -3 gpurun_out/xs2_xattn_live.err
timeout 900 python tools/xattn_bench.py --tau 0.9 > gpurun_out/xs2_bench_tc.json 2> gpurun_out/xs2_bench_tc.err; echo "xb rc=$?"
