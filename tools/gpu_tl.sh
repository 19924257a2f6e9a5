set -x
timeout 300 python tools/bars_fwd.py bars > gpurun_out/bf.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:attn_fwd_kernel --launch-skip 1 -c 1 -o gpurun_out/bars_fwd python tools/bars_fwd.py bars > gpurun_out/bars_ncu.log 2>&1; echo "ncu bars rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:attn_fwd_kernel --launch-skip 1 -c 1 -o gpurun_out/slash_fwd python tools/bars_fwd.py slash > gpurun_out/slash_ncu.log 2>&1; echo "ncu slash rc=$?"
