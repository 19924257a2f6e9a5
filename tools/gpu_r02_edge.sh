set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
timeout 1500 python -m pytest -q -m gpu tests/test_gpu_edge_cases.py tests/test_gpu_index.py tests/test_gpu_attn_fwd.py tests/test_gpu_attn_bwd.py tests/test_gpu_rope_index.py tests/test_gpu_stripe.py > gpurun_out/edge_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/edge_pytest.log
