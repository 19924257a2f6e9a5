set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
timeout 900 python -m pytest -q -m gpu tests/test_gpu_rope_index.py tests/test_gpu_rope.py tests/test_gpu_attn_fwd.py tests/test_gpu_ring.py tests/test_gpu_configs.py tests/test_gpu_env_cases.py > gpurun_out/stab_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/stab_pytest.log
timeout 900 python tools/imbalance_report.py --out gpurun_out/r02_imbalance.json > gpurun_out/stab_imb.log 2>&1; echo "imb rc=$?"; grep measured gpurun_out/stab_imb.log
for lay in striped zigzag; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29634 bench.py --gpus 4 --layout $lay --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/stab_bench_n4_$lay.json 2> gpurun_out/stab_bench_n4_$lay.err; echo "bench n4 $lay rc=$?"
done
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/stab_bench_n1.json 2> gpurun_out/stab_bench_n1.err; echo "bench n1 rc=$?"
