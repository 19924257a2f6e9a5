# merged index sort: bit-exact tests (index, full size, rings on 2 GPUs) + bench lines at C1/C2/C3/C4
set -x
timeout 900 python -m pytest tests/test_gpu_index.py tests/test_gpu_fullsize.py tests/test_gpu_ring.py -q -x > gpurun_out/idx_pytest.log 2>&1; echo "pytest rc=$?"
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --seq 4096 --hq 8 --hkv 1 > gpurun_out/idx_c1.json 2> gpurun_out/idx_c1.err; echo "c1 rc=$?"
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --seq 65536 > gpurun_out/idx_c2.json 2> gpurun_out/idx_c2.err; echo "c2 rc=$?"
timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --seq 131072 > gpurun_out/idx_c3.json 2> gpurun_out/idx_c3.err; echo "c3 rc=$?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/idx_c4.json 2> gpurun_out/idx_c4.err; echo "c4 rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/idx_c4_n2.json 2> gpurun_out/idx_c4_n2.err; echo "c4 n2 rc=$?"
