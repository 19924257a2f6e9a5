#!/bin/bash
# heads per BLOCK tile and Q/dO stage count under the final backward (512K N=1 bwd ms)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -x -m gpu -k "bwd" > gpurun_out/hp_pytest_s3.log 2>&1 || true
for rep in 1 2; do
  for v in h4 h2 h8 s3; do
    d=.; env=""
    case $v in h2) env="MT_BWD_HPT=2";; h8) env="MT_BWD_HPT=8";; s3) d=tools/ab/s3;; esac
    env $env timeout 600 python $d/bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/hp_${v}_$rep.json 2> gpurun_out/hp_${v}_$rep.err
    python -c "import json;d=json.loads(open('gpurun_out/hp_${v}_$rep.json').read().strip().splitlines()[-1]);print('$v',$rep,round(d['value']),d['roofline']['phase_ms'],d['clocks']['sm_mhz'])"
  done
done
