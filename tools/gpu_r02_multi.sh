# round-2 multi-GPU pass: full GPU suite on 4 GPUs, bench at N = 1, 2, 4 (and 2x2), forward timeline
set -x
nvidia-smi -L
python -c "from paper_2510_18830_b200 import build; build.build()"
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r02_pytest_gpu_4gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r02_pytest_gpu_4gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02_multi_n1.json 2> gpurun_out/r02_multi_n1.err; echo "n1 rc=$?"
for n in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $n --steps 10 --warmup 3 > gpurun_out/r02_multi_n$n.json 2> gpurun_out/r02_multi_n$n.err; echo "n$n rc=$?"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 4 --inner 2 --steps 10 --warmup 3 > gpurun_out/r02_multi_n4_2x2.json 2> gpurun_out/r02_multi_n4_2x2.err; echo "2x2 rc=$?"
for f in n1 n2 n4 n4_2x2; do python -c "
import json;d=json.load(open('gpurun_out/r02_multi_$f.json'));r=d['roofline'];print('$f', round(d['value']), d['e2e']['value'] if d.get('e2e') else None, r['phase_ms'], r['frac'], d['clocks']['sm_mhz'])"; done
