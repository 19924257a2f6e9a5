set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
timeout 900 python bench.py --seq 4096 --hq 8 --hkv 1 --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/r02_bench_c1g.json 2> gpurun_out/r02_bench_c1g.err; echo "c1 rc=$?"
timeout 900 python bench.py --seq 65536 --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/r02_bench_c2g.json 2> gpurun_out/r02_bench_c2g.err; echo "c2 rc=$?"
cat gpurun_out/r02_bench_c1g.json gpurun_out/r02_bench_c2g.json; tail -5 gpurun_out/r02_bench_c1g.err
