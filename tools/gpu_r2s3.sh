# session-3 baseline: smoke, gpu tests, bench (ours + reference arm), launch list
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo ref=$?
for f in gpurun_out/bench.log gpurun_out/bench_ref.log gpurun_out/pytest_gpu.log; do tail -n 3 $f; done
