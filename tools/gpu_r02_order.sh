set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
for rep in 1 2; do for o in 1 0; do
MT_FWD_ORDER=$o timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 4 --warmup 3 > gpurun_out/ord_${o}_$rep.json 2>&1; echo "o$o rc=$?"
done; done
M=dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum
for o in 1 0; do
MT_FWD_ORDER=$o timeout 600 ncu --metrics $M --clock-control none -k regex:attn_fwd_kernel -c 1 --csv python tools/prof_step.py --seq 524288 --reps 1 > gpurun_out/ord_ncu_$o.csv 2>&1; echo "ncu $o rc=$?"
done
