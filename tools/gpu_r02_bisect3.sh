set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
for rep in 1 2; do
for c in v0 226bc7c; do
(cd tools/ab/$c && timeout 600 ncu --metrics $M --clock-control none -k regex:attn_bwd_kernel -c 1 --csv python prof_step.py --seq 524288 --reps 1 > ../../../gpurun_out/bis3_${c}_$rep.csv 2>&1); echo "$c rc=$?"
done
timeout 600 ncu --metrics $M --clock-control none -k regex:attn_bwd_kernel -c 1 --csv python tools/prof_step.py --seq 524288 --reps 1 > gpurun_out/bis3_cur_$rep.csv 2>&1; echo "cur rc=$?"
MT_BWD_SPLIT=1 timeout 600 ncu --metrics $M --clock-control none -k regex:attn_bwd_kernel -c 1 --csv python tools/prof_step.py --seq 524288 --reps 1 > gpurun_out/bis3_split_$rep.csv 2>&1; echo "split rc=$?"
done
