# backward knock-outs at 512K (bench phase split): baseline, no dQ reduce, per-element red
set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
for v in 0 1 4; do
  MT_BWD_DBG=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02_bwdab_$v.json 2> gpurun_out/r02_bwdab_$v.err; echo "dbg=$v rc=$?"
done
