# tests + bench + step timeline (CUPTI) after the round-2 attention/pair-barrier changes
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 600 python tools/timeline.py > gpurun_out/timeline.txt 2>&1; echo timeline=$?
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.log".replace("bench.log", "bench.log")).read().splitlines()[-1]) if False else None
PY
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'], d['e2e']['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['roofline_gemm']['frac'], d['roofline_kernel1'], d['clocks'])"
head -40 gpurun_out/timeline.txt
