set -x
timeout 1200 python -m pytest tests/test_gpu_ring.py tests/test_gpu_layer_ring.py -q > gpurun_out/r01v11_multi_pytest.log 2>&1; echo "multi pytest rc=$?"
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 5 --warmup 3 > gpurun_out/r01v11_multi_bench_n$n.json 2> gpurun_out/r01v11_multi_bench_n$n.err; echo "bench n=$n rc=$?"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --inner 2 --steps 5 --warmup 3 > gpurun_out/r01v11_multi_bench_n4_2x2.json 2> gpurun_out/r01v11_multi_bench_n4_2x2.err; echo "bench 2x2 rc=$?"
