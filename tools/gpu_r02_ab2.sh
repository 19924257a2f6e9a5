set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
timeout 900 python -m pytest -q -m gpu tests/test_gpu_attn_fwd.py tests/test_gpu_attn_bwd.py tests/test_gpu_block_sparse.py tests/test_gpu_fullsize.py tests/test_gpu_rope_index.py > gpurun_out/ab2_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/ab2_pytest.log
for rep in 1 2; do
(cd tools/ab/v0 && timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > ../../../gpurun_out/ab2_v0_$rep.json 2>&1); echo "v0 rc=$?"
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/ab2_cur_$rep.json 2>&1; echo "cur rc=$?"
done
timeout 300 python bench.py --seq 4096 --hq 8 --hkv 1 --no-cpu-baseline --no-e2e --steps 20 --warmup 5 > gpurun_out/ab2_c1.json 2>&1; echo "c1 rc=$?"
timeout 300 python tools/live_kernel_times.py --seq 4096 --hq 8 --hkv 1 > gpurun_out/ab2_c1_live.json 2> gpurun_out/ab2_c1_live.err; echo "live rc=$?"
