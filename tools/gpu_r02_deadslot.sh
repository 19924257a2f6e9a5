#!/bin/bash
# dead-slot skips in the backward block pass: A/B on one box (bench 512K N=1) + parity
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ds_build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -q -x -m gpu -k "bwd or edge or ring_local or guard" > gpurun_out/ds_pytest.log 2>&1
tail -3 gpurun_out/ds_pytest.log
for rep in 1 2; do
for dbg in 0 192 64 128; do
  MT_BWD_DBG=$dbg timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ds_dbg${dbg}_$rep.json 2> gpurun_out/ds_dbg${dbg}_$rep.err
  python -c "import json;d=json.loads(open('gpurun_out/ds_dbg${dbg}_$rep.json').read().strip().splitlines()[-1]);print($dbg,$rep,round(d['value']),d['roofline']['phase_ms'],d['roofline']['frac'],d['clocks']['sm_mhz'])"
done
done
