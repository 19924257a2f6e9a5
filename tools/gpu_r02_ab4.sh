set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
timeout 900 python -m pytest -q -m gpu tests/test_gpu_index.py tests/test_gpu_attn_bwd.py tests/test_gpu_env_cases.py tests/test_gpu_configs.py > gpurun_out/ab4_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ab4_pytest.log
for rep in 1 2; do
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/ab4_cur_$rep.json 2>&1; echo "cur rc=$?"
done
(cd tools/ab/v0 && timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > ../../../gpurun_out/ab4_v0.json 2>&1); echo "v0 rc=$?"
timeout 300 python bench.py --seq 4096 --hq 8 --hkv 1 --no-cpu-baseline --no-e2e --steps 20 --warmup 5 > gpurun_out/ab4_c1.json 2>&1; echo "c1 rc=$?"
timeout 300 python tools/live_kernel_times.py --seq 4096 --hq 8 --hkv 1 > gpurun_out/ab4_c1_live.json 2> gpurun_out/ab4_c1_live.err; echo "live rc=$?"
timeout 600 python tools/live_kernel_times.py --seq 524288 --hq 16 --hkv 2 --xattn 0.9 --steps 2 --warmup 1 > gpurun_out/ab4_xattn_live.json 2> gpurun_out/ab4_xattn_live.err; echo "xlive rc=$?"
