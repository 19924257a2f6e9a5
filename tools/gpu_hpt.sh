# backward block pass with several q heads per tile (MT_BWD_HPT): parity + A/B
set -x
for h in 2 4; do
  MT_BWD_HPT=$h timeout 900 python -m pytest tests/test_gpu_attn_bwd.py -q -x > gpurun_out/hpt_pytest_$h.log 2>&1; echo "pytest hpt=$h rc=$?"
done
for rep in a b; do
for h in 1 2 4 8; do
  MT_BWD_HPT=$h timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/hpt_c4_${h}_$rep.json 2> gpurun_out/hpt_c4_${h}_$rep.err; echo "c4 hpt=$h rc=$?"
  MT_BWD_HPT=$h timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --seq 131072 > gpurun_out/hpt_c3_${h}_$rep.json 2> gpurun_out/hpt_c3_${h}_$rep.err; echo "c3 hpt=$h rc=$?"
done
done
