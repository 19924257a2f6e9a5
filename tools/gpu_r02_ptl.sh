set -x
MT_NVCC_EXTRA="-DMT_TIMELINE -DMT_TL_PROD" python -c "from paper_2510_18830_b200 import build; build.build()"
MT_NVCC_EXTRA="-DMT_TIMELINE -DMT_TL_PROD" timeout 600 python tools/fwd_timeline.py 524288 > gpurun_out/r02_fwd_tl_prod.txt 2>&1; echo "tl rc=$?"
python tools/prod_timeline.py 2>&1 || true
python -c "from paper_2510_18830_b200 import build; build.build()"
