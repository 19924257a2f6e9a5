set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
timeout 600 python -m pytest tests/test_gpu_index.py -q -x -k extreme > gpurun_out/r02_pytest_tiny.log 2>&1; echo "tiny rc=$?"; tail -2 gpurun_out/r02_pytest_tiny.log
timeout 900 python bench.py > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err; echo "bench rc=$?"
timeout 900 python bench.py --seq 4096 --hq 8 --hkv 1 --no-cpu-baseline > gpurun_out/r02_bench_c1.json 2> gpurun_out/r02_bench_c1.err; echo "c1 rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_ref.json 2> gpurun_out/r02_bench_ref.err; echo "ref rc=$?"
cat gpurun_out/r02_bench_default.json; cat gpurun_out/r02_bench_c1.json; cat gpurun_out/r02_bench_ref.json
