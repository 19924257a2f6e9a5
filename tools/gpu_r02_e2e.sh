#!/bin/bash
# e2e copy-schedule A/B at N=1 and N=2 (bench.py, 512K)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e2e_build.log 2>&1 || exit 1
for mode in 0 1; do
  MT_BENCH_E2E_EARLY=$mode timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/e2e_n2_early$mode.json 2> gpurun_out/e2e_n2_early$mode.err
done
for mode in 0 1; do
  MT_BENCH_E2E_EARLY=$mode timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/e2e_n1_early$mode.json 2> gpurun_out/e2e_n1_early$mode.err
done
MT_BENCH_E2E_EARLY=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/e2e_n2_s20.json 2> gpurun_out/e2e_n2_s20.err
