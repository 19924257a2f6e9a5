set -x
python -c "from paper_2510_18830_b200 import build; build.build()"
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum
MT_BWD_SPLIT=1 MT_BWD_MEMSET=1 timeout 600 ncu --metrics $M --clock-control none -k regex:attn_bwd_kernel -c 1 --csv python tools/prof_step.py --seq 524288 --reps 1 > gpurun_out/dram_memset.csv 2>&1; echo "memset rc=$?"
MT_BWD_SPLIT=1 timeout 600 ncu --metrics $M --clock-control none -k regex:attn_bwd_kernel -c 1 --csv python tools/prof_step.py --seq 524288 --reps 1 > gpurun_out/dram_split2.csv 2>&1; echo "split rc=$?"
for rep in 1 2; do
MT_BWD_MEMSET=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 4 --warmup 3 > gpurun_out/dram_bench_memset_$rep.json 2>&1; echo "bm rc=$?"
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 4 --warmup 3 > gpurun_out/dram_bench_cur_$rep.json 2>&1; echo "bc rc=$?"
done
