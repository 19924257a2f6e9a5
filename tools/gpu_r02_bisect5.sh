set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_attn_bwd.py tests/test_gpu_edge_cases.py tests/test_gpu_env_cases.py tests/test_gpu_block_sparse.py tests/test_gpu_configs.py tests/test_gpu_fullsize.py > gpurun_out/bis6_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/bis6_pytest.log
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
for rep in 1 2; do
(cd tools/ab/v0 && timeout 600 ncu --metrics $M --clock-control none -k regex:attn_bwd_kernel -c 1 --csv python prof_step.py --seq 524288 --reps 1 > ../../../gpurun_out/bis6_v0_$rep.csv 2>&1); echo "v0 rc=$?"
timeout 600 ncu --metrics $M --clock-control none -k regex:attn_bwd_kernel -c 1 --csv python tools/prof_step.py --seq 524288 --reps 1 > gpurun_out/bis6_split_$rep.csv 2>&1; echo "split rc=$?"
timeout 600 ncu --metrics $M --clock-control none -k regex:attn_bwd_kernel -c 1 --csv python tools/prof_step.py --seq 524288 --reps 1 > gpurun_out/bis6_cur_$rep.csv 2>&1; echo "cur rc=$?"
done
for rep in 1 2; do
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 4 --warmup 3 > gpurun_out/bis6_bench_$rep.json 2>&1; echo "b rc=$?"
(cd tools/ab/v0 && timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 4 --warmup 3 > ../../../gpurun_out/bis6_benchv0_$rep.json 2>&1); echo "bv0 rc=$?"
done
