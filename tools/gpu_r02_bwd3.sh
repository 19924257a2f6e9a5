set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_attn_bwd.py tests/test_gpu_guard.py tests/test_gpu_env_cases.py tests/test_gpu_block_sparse.py -q -x > gpurun_out/r02_bwd3_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02_bwd3_pytest.log
for rep in a b; do
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02_bwd3_bench_$rep.json 2> gpurun_out/r02_bwd3_bench_$rep.err; echo "bench rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/r02_bwd3_bench_$rep.json'));r=d['roofline'];print('3st', round(d['value']), r['phase_ms'], r['frac'], d['clocks']['sm_mhz'])"
done
MT_NVCC_EXTRA="-DMT_BWD_STAGES=4" python -c "from paper_2510_18830_b200 import build; build.build()"
MT_NVCC_EXTRA="-DMT_BWD_STAGES=4" timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02_bwd4_bench.json 2> gpurun_out/r02_bwd4_bench.err; echo "bench4 rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/r02_bwd4_bench.json'));r=d['roofline'];print('4st', round(d['value']), r['phase_ms'], r['frac'], d['clocks']['sm_mhz'])"
