# round-2 closing pass (4-GPU box): every GPU test, smoke, the default bench line, N = 2 / 4 lines, C1,
# the ncu launch list and --set full captures of the backward (both launches) and the forward
set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
P=gpurun_out/${TAG:-r02c}
timeout 1500 python -m pytest tests -m gpu -q > ${P}_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 ${P}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > ${P}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > ${P}_bench.json 2> ${P}_bench.err; echo "bench rc=$?"
timeout 300 python bench.py --seq 4096 --hq 8 --hkv 1 --no-cpu-baseline --steps 20 --warmup 5 > ${P}_c1.json 2> ${P}_c1.err; echo "c1 rc=$?"
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2979$n bench.py --gpus $n --steps 5 --warmup 3 > ${P}_n$n.json 2> ${P}_n$n.err; echo "n$n rc=$?"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29799 bench.py --gpus 4 --inner 2 --steps 5 --warmup 3 > ${P}_n4_2x2.json 2> ${P}_n4_2x2.err; echo "2x2 rc=$?"
CMD='python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline'
timeout 300 $CMD > ${P}_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${P}_launches.csv $CMD > ${P}_ncu_launch.log 2>&1; echo "launches rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:attn_bwd_kernel -c 2 -o ${P}_bwd python tools/prof_step.py --seq 524288 --reps 1 > ${P}_ncu_bwd.log 2>&1; echo "ncu bwd rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_fwd_kernel -c 1 -o ${P}_fwd python tools/prof_step.py --seq 524288 --reps 1 > ${P}_ncu_fwd.log 2>&1; echo "ncu fwd rc=$?"
