# GPU tests, then the multi-process sharded path on a one-GPU box: 2 ranks (torchrun) sharing
# cuda:0 over gloo, and thread-simulated ranks; small configs, hard timeouts, tracebacks on timeout.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
export PYTHONFAULTHANDLER=1 PYTHONUNBUFFERED=1 IFKV_BENCH_WATCHDOG=${WATCHDOG:-140}
SMALL=${SMALL:-"--layers 2 --ctx 4096 --chunk 512 --steps 2 --warmup 1"}
timeout -s ABRT 170 python bench.py --simulate-ranks 2 $SMALL > gpurun_out/sim2.log 2>&1; echo sim rc=$?
tail -1 gpurun_out/sim2.log | cut -c1-400
IFKV_DIST_BACKEND=gloo timeout -s ABRT 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 $SMALL > gpurun_out/dist2_gloo.log 2>&1
echo rc=$?
grep -v "^\s*$" gpurun_out/dist2_gloo.log | grep -v "elastic\|^W1\|^I1" | tail -5 | cut -c1-600
