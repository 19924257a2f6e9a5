set -x
for d in 0 3; do
MT_NVCC_EXTRA="-DMT_TIMELINE -DMT_TL_ISSUER2" python -c "from paper_2510_18830_b200 import build; build.build()"
MT_BWD_DBG=$d MT_NVCC_EXTRA="-DMT_TIMELINE -DMT_TL_ISSUER2" timeout 600 python tools/bwd_timeline_issuer.py 524288 > gpurun_out/r02_tl_issuer_$d.txt 2>&1; echo "tl rc=$?"
cat gpurun_out/r02_tl_issuer_$d.txt
done
