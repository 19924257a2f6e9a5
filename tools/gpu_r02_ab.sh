set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
for rep in 1 2; do
(cd tools/ab/v0 && timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > ../../../gpurun_out/ab_v0_$rep.json 2>&1); echo "v0 rc=$?"
MT_FWD_STABFIX=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/ab_cur1_$rep.json 2>&1; echo "cur1 rc=$?"
MT_FWD_STABFIX=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/ab_cur0_$rep.json 2>&1; echo "cur0 rc=$?"
done
