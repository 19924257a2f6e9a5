# compute-sanitizer (SURVEY §4 test tier v) on small hot-path steps: index + fwd + bwd through the C ABI
# (tools/prof_step.py), C1 shape (S = 4096, 8/1 heads) and a 16/2-head 8K case; writes gpurun_out/r01_san_*
set -x
P=gpurun_out/r01_san
C1='python tools/prof_step.py --seq 4096 --hq 8 --hkv 1 --reps 1'
C2='python tools/prof_step.py --seq 8192 --hq 16 --hkv 2 --reps 1'
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 17 --print-limit 50 $C1 > ${P}_${tool}_c1.log 2>&1
  echo "$tool c1 rc=$?"
done
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 17 --print-limit 50 $C2 > ${P}_memcheck_8k.log 2>&1
echo "memcheck 8k rc=$?"
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 17 --print-limit 50 $C2 > ${P}_racecheck_8k.log 2>&1
echo "racecheck 8k rc=$?"
