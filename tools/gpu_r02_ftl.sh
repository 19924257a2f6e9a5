set -x
MT_NVCC_EXTRA="-DMT_TIMELINE" python -c "from paper_2510_18830_b200 import build; build.build()"
MT_NVCC_EXTRA="-DMT_TIMELINE" timeout 600 python tools/fwd_timeline.py 524288 > gpurun_out/r02_fwd_tl.txt 2>&1; echo "tl rc=$?"
MT_FWD_DBG=1 MT_NVCC_EXTRA="-DMT_TIMELINE" timeout 600 python tools/fwd_timeline.py 524288 > gpurun_out/r02_fwd_tl_nosm.txt 2>&1; echo "tl2 rc=$?"
cat gpurun_out/r02_fwd_tl.txt gpurun_out/r02_fwd_tl_nosm.txt
python -c "from paper_2510_18830_b200 import build; build.build()"
