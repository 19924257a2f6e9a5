set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
timeout 300 python tools/debug_fwd_ring.py 2 2>&1 | tail -5
timeout 900 python -m pytest tests/test_gpu_attn_fwd.py tests/test_gpu_block_sparse.py tests/test_gpu_env_cases.py tests/test_gpu_attn_bwd.py tests/test_gpu_guard.py -q -x > gpurun_out/r02_fwd_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r02_fwd_pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02_fwd_bench.json 2> gpurun_out/r02_fwd_bench.err; echo "bench rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/r02_fwd_bench.json'));r=d['roofline'];print(round(d['value']), r['phase_ms'], r['fwd_tflops'], d['clocks']['sm_mhz'])"
