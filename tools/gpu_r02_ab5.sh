set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
timeout 600 python -m pytest -q -m gpu tests/test_gpu_index.py tests/test_gpu_guard.py > gpurun_out/ab5_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ab5_pytest.log
timeout 300 python tools/live_kernel_times.py --seq 4096 --hq 8 --hkv 1 > gpurun_out/ab5_c1_live.json 2> gpurun_out/ab5_c1_live.err; echo "live rc=$?"
for rep in 1 2; do
(cd tools/ab/v0 && timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 4 --warmup 3 > ../../../gpurun_out/ab5_v0_$rep.json 2>&1); echo "v0 rc=$?"
for d in 0 64 128 192; do
MT_BWD_DBG=$d timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 4 --warmup 3 > gpurun_out/ab5_d${d}_$rep.json 2>&1; echo "d$d rc=$?"
done; done
