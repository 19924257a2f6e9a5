# one-GPU validation + measurement pass (writes gpurun_out/r01v11_*)
set -x
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r01v11_pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r01v11_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r01v11_bench.json 2> gpurun_out/r01v11_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r01v11_bench_ref.json 2> gpurun_out/r01v11_bench_ref.err; echo "ref rc=$?"
CMD='python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline'
timeout 300 $CMD > gpurun_out/r01v11_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01v11_launches.csv $CMD > gpurun_out/r01v11_ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 300 python tools/prof_step.py --seq 524288 --reps 1 > gpurun_out/ps.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:attn_fwd_kernel -c 1 -o gpurun_out/r01v11_fwd python tools/prof_step.py --seq 524288 --reps 1 > gpurun_out/r01v11_ncu_fwd.log 2>&1; echo "ncu fwd rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:attn_bwd_kernel -c 1 -o gpurun_out/r01v11_bwd_block python tools/prof_step.py --seq 524288 --reps 1 > gpurun_out/r01v11_ncu_bwd_block.log 2>&1; echo "ncu bwd block rc=$?"
timeout 1200 ncu --set full --clock-control none -k regex:attn_bwd_kernel --launch-skip 1 -c 1 -o gpurun_out/r01v11_bwd_bar python tools/prof_step.py --seq 524288 --reps 1 > gpurun_out/r01v11_ncu_bwd_bar.log 2>&1; echo "ncu bwd bar rc=$?"
