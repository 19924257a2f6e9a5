# round-2 second final pass (4-GPU box): every GPU test, smoke, default bench line (e2e + cpu_baseline),
# N = 2 / 4 bench lines, C1; TAG prefixes the outputs under gpurun_out/
set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
P=gpurun_out/${TAG:-r02b}
timeout 1500 python -m pytest tests -m gpu -q > ${P}_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 ${P}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > ${P}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > ${P}_bench.json 2> ${P}_bench.err; echo "bench rc=$?"
timeout 300 python bench.py --seq 4096 --hq 8 --hkv 1 --no-cpu-baseline --steps 20 --warmup 5 > ${P}_c1.json 2> ${P}_c1.err; echo "c1 rc=$?"
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2978$n bench.py --gpus $n --steps 5 --warmup 3 > ${P}_n$n.json 2> ${P}_n$n.err; echo "n$n rc=$?"
done
