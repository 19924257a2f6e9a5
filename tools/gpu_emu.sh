# slow inter-node link emulation: 4 GPUs as 2 nodes x 2, flat vs hierarchical ring
set -x
for g in 8; do
  MT_EMU_INTER_GBPS=$g MT_EMU_NODE=2 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 4 --steps 3 --warmup 2 --no-e2e > gpurun_out/emu_flat_$g.json 2> gpurun_out/emu_flat_$g.err; echo "flat rc=$?"
  MT_EMU_INTER_GBPS=$g MT_EMU_NODE=2 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 4 --inner 2 --steps 3 --warmup 2 --no-e2e > gpurun_out/emu_hier_$g.json 2> gpurun_out/emu_hier_$g.err; echo "hier rc=$?"
done
