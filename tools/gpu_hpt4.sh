# MT_BWD_HPT at N = 2 / 4: real-NCCL ring parity + A/B
set -x
MT_BWD_HPT=4 timeout 900 python -m pytest tests/test_gpu_ring.py -q -x > gpurun_out/hpt4_ring_pytest.log 2>&1; echo "ring pytest hpt=4 rc=$?"
run() {  # name n hpt args
  name=$1; n=$2; h=$3; shift 3
  MT_BWD_HPT=$h timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29540 + RANDOM % 300)) bench.py --gpus $n --steps 5 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/hpt4_$name.json 2> gpurun_out/hpt4_$name.err; echo "$name rc=$?"
}
for rep in a b; do
  for h in 1 2 4; do
    run c4_n4_h${h}_$rep 4 $h
    run c3_n4_h${h}_$rep 4 $h --seq 131072
  done
done
for h in 1 4; do run c4_n2_h$h 2 $h; done
