set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_attn_fwd.py tests/test_gpu_env_cases.py tests/test_gpu_block_sparse.py > gpurun_out/pf_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pf_pytest.log
for rep in 1 2; do
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 4 --warmup 3 > gpurun_out/pf_cur_$rep.json 2>&1; echo "cur rc=$?"
(cd tools/ab/v0 && timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 4 --warmup 3 > ../../../gpurun_out/pf_v0_$rep.json 2>&1); echo "v0 rc=$?"
done
