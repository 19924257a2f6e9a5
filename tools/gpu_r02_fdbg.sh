set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
for d in 0 1; do
MT_FWD_DBG=$d timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 4 --warmup 3 > gpurun_out/fdbg_$d.json 2>&1; echo "d$d rc=$?"
done
MT_FWD_DBG=1 MT_BWD_DBG=3 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 4 --warmup 3 > gpurun_out/fdbg_both.json 2>&1; echo "both rc=$?"
