# backward clock64 timelines (CTA 0) at 512K: default, issuer view, WG split; plus no-dQ-reduce
set -x
for v in "" "-DMT_TL_ISSUER" "-DMT_TL_WGSPLIT"; do
  MT_NVCC_EXTRA="-DMT_TIMELINE $v" python -c "from paper_2510_18830_b200 import build; build.build()"
  a=""; [ "$v" = "-DMT_TL_ISSUER" ] && a="--issuer"; [ "$v" = "-DMT_TL_WGSPLIT" ] && a="--wgsplit"
  MT_NVCC_EXTRA="-DMT_TIMELINE $v" timeout 600 python tools/bwd_timeline.py 524288 $a > gpurun_out/r02_tl$v.txt 2>&1; echo "tl $v rc=$?"
  MT_BWD_DBG=1 MT_NVCC_EXTRA="-DMT_TIMELINE $v" timeout 600 python tools/bwd_timeline.py 524288 $a > gpurun_out/r02_tl_dbg1$v.txt 2>&1; echo "tl dbg1 $v rc=$?"
done
