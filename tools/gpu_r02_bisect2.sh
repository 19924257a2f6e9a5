set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum
for d in 0 64 128 192; do
MT_BWD_DBG=$d timeout 600 ncu --metrics $M --clock-control none -k regex:attn_bwd_kernel -c 1 --csv python tools/prof_step.py --seq 524288 --reps 1 > gpurun_out/bis2_d$d.csv 2>&1; echo "d$d rc=$?"
done
