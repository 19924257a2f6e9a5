# f3 validation: rope + layer parity, layer bench at 512K
set -x
timeout 900 python -m pytest tests/test_gpu_rope.py tests/test_gpu_layer.py -q > gpurun_out/f3_pytest.log 2>&1; echo "pytest rc=$?"
timeout 900 python tools/layer_bench.py > gpurun_out/f3_layer_bench.json 2> gpurun_out/f3_layer_bench.err; echo "layer bench rc=$?"
