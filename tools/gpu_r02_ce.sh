# copy-engine ring: real multi-GPU ring tests (plain run = copy engines, guarded = NCCL), bench A/B
set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
timeout 1200 python -m pytest tests/test_gpu_ring.py -q -x -s > gpurun_out/r02_ce_ring.log 2>&1; echo "ring rc=$?"
grep -E "world|passed|failed|Error" gpurun_out/r02_ce_ring.log | head -20
for n in 2 4; do
for ce in 1 0; do
MT_RING_CE=$ce timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2952$n bench.py --gpus $n --steps 10 --warmup 3 --no-e2e > gpurun_out/r02_ce_n${n}_$ce.json 2> gpurun_out/r02_ce_n${n}_$ce.err; echo "n$n ce$ce rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/r02_ce_n${n}_$ce.json'));r=d['roofline'];rg=d.get('ring',{}).get('passes',{}).get('fwd',{})
print('n$n ce$ce', round(d['value']), r['phase_ms'], rg.get('compute_ms_median'), rg.get('kv_ms_median'), rg.get('kv_gbps_best'))"
done
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 4 --seq 131072 --steps 10 --warmup 3 --no-e2e > gpurun_out/r02_ce_c3_n4.json 2> gpurun_out/r02_ce_c3_n4.err; echo "c3 rc=$?"
MT_RING_CE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 4 --seq 131072 --steps 10 --warmup 3 --no-e2e > gpurun_out/r02_ce_c3_n4_nccl.json 2> gpurun_out/r02_ce_c3_n4_nccl.err; echo "c3 nccl rc=$?"
for f in r02_ce_c3_n4 r02_ce_c3_n4_nccl; do python -c "
import json;d=json.load(open('gpurun_out/$f.json'));r=d['roofline'];rg=d.get('ring',{}).get('passes',{}).get('fwd',{})
print('$f', round(d['value']), r['phase_ms'], rg.get('compute_ms_median'), rg.get('kv_ms_median'), rg.get('kv_gbps_best'))"; done
