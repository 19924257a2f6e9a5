set -x
timeout 900 python -m pytest tests/test_gpu_attn_fwd.py tests/test_gpu_attn_bwd.py tests/test_gpu_fullsize.py tests/test_gpu_block_sparse.py -q -x > gpurun_out/pack_pytest.log 2>&1; echo "tests rc=$?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/pack_on.json 2> gpurun_out/pack_on.err; echo "on rc=$?"
MT_FWD_PACK=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/pack_off.json 2> gpurun_out/pack_off.err; echo "off rc=$?"
timeout 600 python tools/split_probe.py > gpurun_out/pack_split.json 2> gpurun_out/pack_split.err; echo "split rc=$?"
