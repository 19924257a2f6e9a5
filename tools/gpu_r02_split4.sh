#!/bin/bash
# N=4: one mixed backward launch per ring step (default at nloc = 2048) vs block-only + bar-only
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/sp_build.log 2>&1 || exit 1
for rep in 1 2; do
for sp in -1 1; do
  MT_BWD_SPLIT=$sp timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2952$rep bench.py --gpus 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sp4_${sp}_$rep.json 2> gpurun_out/sp4_${sp}_$rep.err
  python -c "import json;d=json.loads(open('gpurun_out/sp4_${sp}_$rep.json').read().strip().splitlines()[-1]);print('split',$sp,$rep,round(d['value']),d['roofline']['phase_ms'],d['clocks']['sm_mhz'])"
done
done
