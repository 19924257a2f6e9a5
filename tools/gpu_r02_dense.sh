set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
timeout 900 python tools/dense_bench.py --steps 2 --warmup 1 > gpurun_out/r02_dense_n1.jsonl 2> gpurun_out/r02_dense_n1.err; echo "n1 rc=$?"
cat gpurun_out/r02_dense_n1.jsonl
for n in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2954$n tools/dense_bench.py --steps 2 --warmup 1 > gpurun_out/r02_dense_n$n.jsonl 2> gpurun_out/r02_dense_n$n.err; echo "n$n rc=$?"
cat gpurun_out/r02_dense_n$n.jsonl
done
timeout 300 python bench.py --seq 4096 --hq 8 --hkv 1 --no-cpu-baseline --no-e2e --graph off --steps 3 --warmup 3 > gpurun_out/c1_plain.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 60 -c 60 --csv --log-file gpurun_out/r02_c1_launches.csv python bench.py --seq 4096 --hq 8 --hkv 1 --no-cpu-baseline --no-e2e --graph off --steps 3 --warmup 3 > gpurun_out/c1_ncu.log 2>&1; echo "ncu rc=$?"
