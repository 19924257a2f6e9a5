set -x
for T in 0.5 0.3 0.15; do
timeout 900 python tools/xattn_bench.py --tau $T --steps 2 > gpurun_out/f2_xattn_bench_$T.json 2> gpurun_out/f2_xattn_bench_$T.err; echo "xbench $T rc=$?"
done
