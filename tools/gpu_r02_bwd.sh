# backward check: parity tests, then the bench line with both dQ paths
set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_attn_bwd.py tests/test_gpu_guard.py -q -x > gpurun_out/r02_bwd_pytest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02_bwd_pytest.log
for red in 0 1; do
MT_BWD_DQ_RED=$red timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02_bwd_bench_$red.json 2> gpurun_out/r02_bwd_bench_$red.err; echo "bench rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/r02_bwd_bench_$red.json'));r=d['roofline'];print('red=$red', round(d['value']), r['phase_ms'], r['frac'], d['clocks']['sm_mhz'])"
done
