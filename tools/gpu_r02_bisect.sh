set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum
for c in v0 62c33c2 226bc7c; do
(cd tools/ab/$c && timeout 600 ncu --metrics $M --clock-control none -k regex:attn_bwd_kernel -c 1 --csv python prof_step.py --seq 524288 --reps 1 > ../../../gpurun_out/bis_$c.csv 2>&1); echo "$c rc=$?"
done
timeout 600 ncu --metrics $M --clock-control none -k regex:attn_bwd_kernel -c 1 --csv python tools/prof_step.py --seq 524288 --reps 1 > gpurun_out/bis_cur.csv 2>&1; echo "cur rc=$?"
