# forward stage-depth A/B: (K 2, V 3) prebuilt vs (K 3, V 2) rebuilt on the box
set -x
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/fab_k2v3.json 2> gpurun_out/fab_k2v3.err; echo "a rc=$?"
MT_NVCC_EXTRA="-DMT_FWD_KST=3 -DMT_FWD_VST=2" timeout 900 python -c "import sys; sys.path.insert(0,'.'); from paper_2510_18830_b200 import build; build.build()" > gpurun_out/fab_build.log 2>&1; echo "build rc=$?"
MT_NVCC_EXTRA="-DMT_FWD_KST=3 -DMT_FWD_VST=2" timeout 900 python -m pytest tests/test_gpu_attn_fwd.py -q -x > gpurun_out/fab_k3v2_pytest.log 2>&1; echo "fwd tests rc=$?"
MT_NVCC_EXTRA="-DMT_FWD_KST=3 -DMT_FWD_VST=2" timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/fab_k3v2.json 2> gpurun_out/fab_k3v2.err; echo "b rc=$?"
MT_NVCC_EXTRA="-DMT_FWD_KST=3 -DMT_FWD_VST=2" timeout 900 python tools/split_probe.py > gpurun_out/fab_k3v2_split.json 2>&1; echo "split rc=$?"
