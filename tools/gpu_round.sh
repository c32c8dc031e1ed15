set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo ref=$?
for f in gpurun_out/bench.log gpurun_out/bench_ref.log gpurun_out/pytest_gpu.log; do tail -n 3 $f; done
