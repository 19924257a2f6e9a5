# backward rewrite check: parity tests, then the bench line
set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_attn_bwd.py tests/test_gpu_guard.py -q -x > gpurun_out/r02_bwd_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02_bwd_pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02_bwd_bench.json 2> gpurun_out/r02_bwd_bench.err; echo "bench rc=$?"
cat gpurun_out/r02_bwd_bench.json | head -c 600
