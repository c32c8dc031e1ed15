# Full C2 size, 2 ranks over gloo sharing cuda:0 (functional check of the torchrun path at scale).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
export PYTHONFAULTHANDLER=1 PYTHONUNBUFFERED=1 IFKV_BENCH_WATCHDOG=420
IFKV_DIST_BACKEND=gloo timeout -s ABRT 480 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 2 --steps 2 --warmup 1 > gpurun_out/dist2_full.log 2>&1
echo rc=$?
grep -v "^\s*$" gpurun_out/dist2_full.log | grep -v "elastic\|^W1\|^I1" | tail -4 | cut -c1-1200
