set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
timeout 1500 python -m pytest -q -x -m gpu tests > gpurun_out/c1_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/c1_pytest.log
timeout 300 python bench.py --seq 4096 --hq 8 --hkv 1 --no-cpu-baseline --no-e2e --steps 20 --warmup 5 > gpurun_out/c1_bench.json 2>&1; echo "c1 rc=$?"
timeout 300 python tools/live_kernel_times.py --seq 4096 --hq 8 --hkv 1 > gpurun_out/c1_live.json 2> gpurun_out/c1_live.err; echo "live rc=$?"
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/c1_512k.json 2> gpurun_out/c1_512k.err; echo "512k rc=$?"
