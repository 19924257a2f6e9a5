set -x
MT_NVCC_EXTRA="-DMT_TIMELINE" python -c "from paper_2510_18830_b200 import build; build.build()"
MT_NVCC_EXTRA="-DMT_TIMELINE" timeout 600 python tools/bwd_timeline2.py 524288 > gpurun_out/r02_tl_pair.txt 2>&1; echo "tl rc=$?"
MT_BWD_DBG=3 MT_NVCC_EXTRA="-DMT_TIMELINE" timeout 600 python tools/bwd_timeline2.py 524288 > gpurun_out/r02_tl_pair_dbg3.txt 2>&1; echo "tl rc=$?"
cat gpurun_out/r02_tl_pair.txt gpurun_out/r02_tl_pair_dbg3.txt
