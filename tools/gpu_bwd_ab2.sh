# backward knock-outs (round-2 kernel): 0 none, 1 no dQ reduce, 2 no softmax, 3 both, 16 no dQ^T MMA, 19 all
set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
for v in 0 1 2 3 16 19; do
  MT_BWD_DBG=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02_bwdab2_$v.json 2> gpurun_out/r02_bwdab2_$v.err; echo "dbg=$v rc=$?"
done
for v in 0 1 2 3 16 19; do python -c "
import json;d=json.load(open('gpurun_out/r02_bwdab2_$v.json'));r=d['roofline'];print($v, r['phase_ms'], d['clocks']['sm_mhz'])"; done
