#!/bin/bash
# A/B: tools/ab/base (prebuilt) vs the working tree (512K N=1 bench, alternating), + bwd parity
mkdir -p gpurun_out
TAG=${TAG:-ab}
timeout 900 python -m pytest tests -q -x -m gpu -k "${PYK:-bwd or edge or guard}" > gpurun_out/${TAG}_pytest.log 2>&1
tail -2 gpurun_out/${TAG}_pytest.log
for rep in 1 2; do
  for v in base new; do
    d=.; [ $v = base ] && d=tools/ab/base
    timeout 600 python $d/bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $EXTRA > gpurun_out/${TAG}_${v}_$rep.json 2> gpurun_out/${TAG}_${v}_$rep.err
    python -c "import json;d=json.loads(open('gpurun_out/${TAG}_${v}_$rep.json').read().strip().splitlines()[-1]);print('$v',$rep,round(d['value']),d['roofline']['phase_ms'],d['clocks']['sm_mhz'])"
  done
done
