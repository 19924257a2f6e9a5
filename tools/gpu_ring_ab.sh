# ring run-ahead: correctness (real NCCL rings) + A/B at N = 4 (MT_RING_AHEAD)
set -x
timeout 900 python -m pytest tests/test_gpu_ring.py tests/test_gpu_layer_ring.py -q -x > gpurun_out/ahead_pytest.log 2>&1; echo "ring tests rc=$?"
run() {  # name, n, env...
  name=$1; n=$2; shift 2
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29530 + RANDOM % 300)) bench.py --gpus $n --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_$name.json 2> gpurun_out/ab_$name.err; echo "$name rc=$?"
}
run n4_ahead 4 MT_RING_AHEAD=1
run n4_old 4 MT_RING_AHEAD=0
run n4_ahead2 4 MT_RING_AHEAD=1
run n4_old2 4 MT_RING_AHEAD=0
