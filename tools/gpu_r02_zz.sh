set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
timeout 1800 python -m pytest -q -m gpu tests > gpurun_out/zz_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/zz_pytest.log
timeout 300 python bench.py --seq 4096 --hq 8 --hkv 1 --no-cpu-baseline --no-e2e --steps 20 --warmup 5 > gpurun_out/zz_c1_bench.json 2>&1; echo "c1 rc=$?"
timeout 300 python tools/live_kernel_times.py --seq 4096 --hq 8 --hkv 1 > gpurun_out/zz_c1_live.json 2> gpurun_out/zz_c1_live.err; echo "live rc=$?"
for n in 4 2; do for lay in striped zigzag; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n bench.py --gpus $n --layout $lay --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/zz_bench_n${n}_$lay.json 2> gpurun_out/zz_bench_n${n}_$lay.err; echo "bench n$n $lay rc=$?"
done; done
timeout 900 python tools/imbalance_report.py --out gpurun_out/r02_imbalance.json > gpurun_out/zz_imb.log 2>&1; echo "imb rc=$?"; tail -30 gpurun_out/zz_imb.log
