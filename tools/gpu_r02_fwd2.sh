set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_attn_fwd.py tests/test_gpu_block_sparse.py tests/test_gpu_env_cases.py -q -x > gpurun_out/r02_fwd_pytest.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/r02_fwd_pytest.log
MT_NVCC_EXTRA="-DMT_TIMELINE" python -c "from paper_2510_18830_b200 import build; build.build()"
MT_NVCC_EXTRA="-DMT_TIMELINE" timeout 600 python tools/fwd_timeline.py 524288 > gpurun_out/r02_fwd_tl.txt 2>&1; echo "tl rc=$?"
cat gpurun_out/r02_fwd_tl.txt
