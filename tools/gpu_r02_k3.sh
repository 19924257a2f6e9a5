set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
for rep in 1 2; do
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 4 --warmup 3 > gpurun_out/k3_base_$rep.json 2>&1; echo "base rc=$?"
done
cp paper_2510_18830_b200/libmtsa.so /tmp/libmtsa_base.so
MT_NVCC_EXTRA="-DMT_FWD_KST=3 -DMT_FWD_VST=2" timeout 900 python -c "from paper_2510_18830_b200 import build; build.build()" > gpurun_out/k3_build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_attn_fwd.py -q -x -m gpu > gpurun_out/k3_pytest.log 2>&1; echo "fwd tests rc=$?"; tail -2 gpurun_out/k3_pytest.log
for rep in 1 2; do
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 4 --warmup 3 > gpurun_out/k3_k3v2_$rep.json 2>&1; echo "k3 rc=$?"
done
