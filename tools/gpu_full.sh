# one-GPU validation + measurement pass (writes gpurun_out/r01v4_*)
set -x
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r01v4_pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r01v4_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r01v4_bench.json 2> gpurun_out/r01v4_bench.err; echo "bench rc=$?"
CMD='python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline'
timeout 300 $CMD > gpurun_out/r01v4_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01v4_launches.csv $CMD > gpurun_out/r01v4_ncu_launch.log 2>&1; echo "launches rc=$?"
timeout 300 python tools/prof_step.py --seq 524288 --reps 1 > gpurun_out/ps.log 2>&1 && timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"attn_(fwd|bwd)_kernel" -c 3 -o gpurun_out/r01v4_attn_full python tools/prof_step.py --seq 524288 --reps 1 > gpurun_out/r01v4_ncu_full.log 2>&1; echo "ncu full rc=$?"
