set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_attn_bwd.py tests/test_gpu_env_cases.py tests/test_gpu_configs.py tests/test_gpu_block_sparse.py tests/test_gpu_fullsize.py > gpurun_out/merge_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/merge_pytest.log
for bf in 1 0; do
MT_BWD_BAR_FIRST=$bf timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/merge_512k_bf$bf.json 2> gpurun_out/merge_512k_bf$bf.err; echo "512k bf$bf rc=$?"
MT_BWD_BAR_FIRST=$bf timeout 300 python bench.py --seq 4096 --hq 8 --hkv 1 --no-cpu-baseline --no-e2e --steps 20 --warmup 5 > gpurun_out/merge_c1_bf$bf.json 2>&1; echo "c1 bf$bf rc=$?"
MT_BWD_BAR_FIRST=$bf timeout 300 python bench.py --seq 131072 --no-cpu-baseline --no-e2e --steps 10 --warmup 3 > gpurun_out/merge_c3_bf$bf.json 2>&1; echo "c3 bf$bf rc=$?"
done
MT_BWD_BAR_PART=1024 timeout 300 python bench.py --seq 4096 --hq 8 --hkv 1 --no-cpu-baseline --no-e2e --steps 20 --warmup 5 > gpurun_out/merge_c1_p1024.json 2>&1; echo "c1 p1024 rc=$?"
MT_BWD_HPT=4 timeout 300 python bench.py --seq 131072 --no-cpu-baseline --no-e2e --steps 10 --warmup 3 > gpurun_out/merge_c3_p1024.json 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 60 --csv --log-file gpurun_out/r02_c1_launches_merge.csv python bench.py --seq 4096 --hq 8 --hkv 1 --no-cpu-baseline --no-e2e --graph off --steps 3 --warmup 3 > gpurun_out/c1_ncu.log 2>&1; echo "ncu rc=$?"
