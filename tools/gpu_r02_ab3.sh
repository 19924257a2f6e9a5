set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
for rep in 1 2; do
for v in "cur:" "split:MT_BWD_SPLIT=1" "red1:MT_BWD_DBG=32" "both:MT_BWD_SPLIT=1 MT_BWD_DBG=32"; do
name=${v%%:*}; envs=${v#*:}
env $envs timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > gpurun_out/ab3_${name}_$rep.json 2>&1; echo "$name rc=$?"
done; done
(cd tools/ab/v0 && timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 5 --warmup 3 > ../../../gpurun_out/ab3_v0.json 2>&1); echo "v0 rc=$?"
