set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
timeout 300 python tools/debug_fwd_ring.py 2 2>&1 | tail -6
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02_fwd_bench.json 2> gpurun_out/r02_fwd_bench.err; echo "bench rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/r02_fwd_bench.json'));r=d['roofline'];print(round(d['value']), r['phase_ms'], r['fwd_tflops'], d['clocks']['sm_mhz'])"
