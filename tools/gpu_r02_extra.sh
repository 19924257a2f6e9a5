#!/bin/bash
# final-code extras: the default bench at 20 steps, zigzag rings at N = 2 / 4
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/x_build.log 2>&1 || exit 1
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r02f_bench_s20.json 2> gpurun_out/x_s20.err; echo "s20 rc=$?"
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2988$n bench.py --gpus $n --layout zigzag --steps 5 --warmup 3 > gpurun_out/r02f_n${n}_zigzag.json 2> gpurun_out/x_zz$n.err; echo "zz$n rc=$?"
done
