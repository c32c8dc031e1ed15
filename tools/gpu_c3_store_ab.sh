set -x
timeout 900 python -m pytest tests/test_gpu_path.py -x -q -m gpu -k "reorder" > gpurun_out/c3_tests.log 2>&1; tail -3 gpurun_out/c3_tests.log
timeout 900 python -m pytest tests/test_gpu_headline.py -x -q -m gpu -k "c3 or reorder" > gpurun_out/c3_headline.log 2>&1; tail -3 gpurun_out/c3_headline.log
for r in 1 2; do
for v in 1 0; do
IFKV_FIRST_PASS_STORE=$v timeout 600 python bench.py --reorder --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-sdpa-comparator > gpurun_out/c3_store$v.$r.log 2>&1
tail -1 gpurun_out/c3_store$v.$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("store='$v'", round(d["ms_per_step"],2), d["stages_ms"], d["clocks"]["sm_mhz"])'
done; done
