# every BASELINE.json config on one 4-GPU box: C1 (4K, 8/1 heads), C2 (64K), C3 (128K at 1/2/4),
# C5 (1M, flat vs 2x2 at 4 GPUs; 8 GPUs are not offered by gpurun). Device numbers, --no-e2e.
set -x
one() {  # name, n, args...
  name=$1; n=$2; shift 2
  if [ "$n" = 1 ]; then
    timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/cfg_$name.json 2> gpurun_out/cfg_$name.err
  else
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29540 + RANDOM % 300)) bench.py --gpus $n --steps 5 --warmup 3 --no-e2e --no-cpu-baseline "$@" \
      > gpurun_out/cfg_$name.json 2> gpurun_out/cfg_$name.err
  fi
  echo "$name rc=$?"
}
one c1 1 --seq 4096 --hq 8 --hkv 1
one c2 1 --seq 65536
one c3_n1 1 --seq 131072
one c3_n2 2 --seq 131072
one c3_n4 4 --seq 131072
one c3_n4_2x2 4 --seq 131072 --inner 2
one c5_n1 1 --seq 1048576
one c5_n4 4 --seq 1048576
one c5_n4_2x2 4 --seq 1048576 --inner 2
