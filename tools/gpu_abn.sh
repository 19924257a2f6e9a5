#!/bin/bash
# A/B over tools/ab/<variant> dirs (prebuilt) and the working tree ("new"), 512K N=1 bench, alternating
mkdir -p gpurun_out
TAG=${TAG:-abn}
VARS=${VARS:-base new}
for rep in 1 2; do
  for v in $VARS; do
    d=.; [ $v != new ] && d=tools/ab/$v
    timeout 600 python $d/bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_${v}_$rep.json 2> gpurun_out/${TAG}_${v}_$rep.err
    python -c "import json;d=json.loads(open('gpurun_out/${TAG}_${v}_$rep.json').read().strip().splitlines()[-1]);print('$v',$rep,round(d['value']),d['roofline']['phase_ms'],d['clocks']['sm_mhz'])"
  done
done
