set -x
MT_FWD_ORDER=0 timeout 600 python tools/split_probe.py > gpurun_out/split_order0.json 2> gpurun_out/split_order0.err; echo "order0 rc=$?"
MT_FWD_ORDER=1 timeout 600 python tools/split_probe.py > gpurun_out/split_order1.json 2> gpurun_out/split_order1.err; echo "order1 rc=$?"
