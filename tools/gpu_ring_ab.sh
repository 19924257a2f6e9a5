# A/B of the SM reservation for NCCL in ring mode (MT_RING_RESERVE_SMS[_BWD]) and CE P2P
set -x
run() {  # name, n, env...
  name=$1; n=$2; shift 2
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29530 + RANDOM % 300)) bench.py --gpus $n --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_$name.json 2> gpurun_out/ab_$name.err; echo "$name rc=$?"
}
for n in 2 4; do
  run n${n}_base $n MT_RING_RESERVE_SMS=0
  run n${n}_f8 $n MT_RING_RESERVE_SMS=8
  run n${n}_f6 $n MT_RING_RESERVE_SMS=6
  run n${n}_ce $n MT_RING_RESERVE_SMS=0 NCCL_P2P_USE_CUDA_MEMCPY=1
  run n${n}_base2 $n MT_RING_RESERVE_SMS=0
done
