# f2 validation: block-CSR attention parity (+ later the XAttention index)
set -x
timeout 900 python -m pytest tests/test_gpu_block_sparse.py -q -x > gpurun_out/f2_pytest.log 2>&1; echo "pytest rc=$?"
if ls tests/test_gpu_xattn.py >/dev/null 2>&1; then timeout 900 python -m pytest tests/test_gpu_xattn.py -q -x > gpurun_out/f2_xattn.log 2>&1; echo "xattn rc=$?"; fi
if [ -n "$F2_BENCH" ]; then timeout 900 python bench.py --no-cpu-baseline > gpurun_out/f2_bench.json 2> gpurun_out/f2_bench.err; echo "bench rc=$?"; fi
