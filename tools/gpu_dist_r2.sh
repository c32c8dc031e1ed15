# sharded path on a one-GPU box with the final library: thread-simulated ranks,
# 2 torchrun processes over gloo at a small and at the full C2 size, and the
# 2-process TorchComm GPU test
export PYTHONFAULTHANDLER=1 PYTHONUNBUFFERED=1 IFKV_BENCH_WATCHDOG=300
SMALL="--layers 2 --ctx 4096 --chunk 512 --steps 2 --warmup 1"
timeout -s ABRT 300 python bench.py --simulate-ranks 2 $SMALL > gpurun_out/sim2.log 2>&1; echo sim rc=$?
tail -1 gpurun_out/sim2.log | cut -c1-300
IFKV_DIST_BACKEND=gloo timeout -s ABRT 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 $SMALL > gpurun_out/dist2_gloo.log 2>&1
echo dist_small rc=$?
grep '^{' gpurun_out/dist2_gloo.log | tail -1 | cut -c1-400
IFKV_DIST_BACKEND=gloo timeout -s ABRT 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 2 --steps 2 --warmup 3 > gpurun_out/dist2_full.log 2>&1
echo dist_full rc=$?
grep '^{' gpurun_out/dist2_full.log | tail -1 | cut -c1-500
timeout 600 python -m pytest tests/test_gpu_sharding.py -q -m gpu -p no:cacheprovider > gpurun_out/pytest_shard.log 2>&1; echo shard_tests=$?
tail -1 gpurun_out/pytest_shard.log
