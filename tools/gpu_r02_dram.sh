set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:attn_bwd_kernel -c 1 --csv python tools/prof_step.py --seq 524288 --reps 1 > gpurun_out/dram_cur.csv 2>&1; echo "cur rc=$?"
MT_BWD_SPLIT=1 timeout 600 ncu --metrics $M --clock-control none -k regex:attn_bwd_kernel -c 2 --csv python tools/prof_step.py --seq 524288 --reps 1 > gpurun_out/dram_split.csv 2>&1; echo "split rc=$?"
(cd tools/ab/v0 && timeout 600 ncu --metrics $M --clock-control none -k regex:attn_bwd_kernel -c 2 --csv python prof_step.py --seq 524288 --reps 1 > ../../../gpurun_out/dram_v0.csv 2>&1); echo "v0 rc=$?"
