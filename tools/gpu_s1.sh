# index stage 1 register tiling: bit-exact tests for both variants + A/B of the index phase
set -x
timeout 900 python -m pytest tests/test_gpu_index.py tests/test_gpu_fullsize.py -q -x > gpurun_out/s1_pytest.log 2>&1; echo "pytest minb3 rc=$?"
MT_VS_S1_MINB=2 timeout 900 python -m pytest tests/test_gpu_index.py -q -x -k "bitexact" > gpurun_out/s1_pytest2.log 2>&1; echo "pytest minb2 rc=$?"
for v in 3 2 3 2; do
  MT_VS_S1_MINB=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s1_c4_$v.json 2> gpurun_out/s1_c4_$v.err; echo "c4 $v rc=$?"
  MT_VS_S1_MINB=$v timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --seq 65536 > gpurun_out/s1_c2_$v.json 2> gpurun_out/s1_c2_$v.err; echo "c2 $v rc=$?"
done
