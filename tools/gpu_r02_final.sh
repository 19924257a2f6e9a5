# round-2 final pass on one 4-GPU box (writes gpurun_out/$TAG_*): every GPU test (incl. 2/4-GPU rings),
# smoke, the default bench line (e2e + cpu_baseline), the reference arm, the ncu launch list, and every
# BASELINE config (C1-C5) at 1/2/4 GPUs, flat and 2x2.
set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
P=gpurun_out/${TAG:-r02a}
timeout 1500 python -m pytest tests -m gpu -q > ${P}_pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > ${P}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > ${P}_bench.json 2> ${P}_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > ${P}_bench_ref.json 2> ${P}_bench_ref.err; echo "ref rc=$?"
CMD='python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline'
timeout 300 $CMD > ${P}_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${P}_launches.csv $CMD > ${P}_ncu_launch.log 2>&1; echo "launches rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_bwd_kernel -c 1 -o ${P}_bwd_block python tools/prof_step.py --seq 524288 --reps 1 > ${P}_ncu_bwd_block.log 2>&1; echo "ncu bwd block rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_fwd_kernel -c 1 -o ${P}_fwd python tools/prof_step.py --seq 524288 --reps 1 > ${P}_ncu_fwd.log 2>&1; echo "ncu fwd rc=$?"
one() {  # name, n, args...
  name=$1; n=$2; shift 2
  if [ "$n" = 1 ]; then
    timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline "$@" > ${P}_cfg_$name.json 2> ${P}_cfg_$name.err
  else
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29540 + RANDOM % 300)) bench.py --gpus $n --steps 5 --warmup 3 "$@" \
      > ${P}_cfg_$name.json 2> ${P}_cfg_$name.err
  fi
  echo "$name rc=$?"
}
one c4_n2 2
one c4_n4 4
one c4_n4_2x2 4 --inner 2
one c1 1 --seq 4096 --hq 8 --hkv 1
one c2 1 --seq 65536
one c3_n1 1 --seq 131072
one c3_n2 2 --seq 131072
one c3_n4 4 --seq 131072
one c3_n4_2x2 4 --seq 131072 --inner 2
one c5_n1 1 --seq 1048576 --no-e2e
one c5_n4 4 --seq 1048576
one c5_n4_2x2 4 --seq 1048576 --inner 2
one c4_n4_zigzag 4 --layout zigzag
one c4_n2_zigzag 2 --layout zigzag
