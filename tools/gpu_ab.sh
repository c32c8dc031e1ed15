# tests + A/B bench runs: bash tools/gpu_ab.sh "ENV=a" "ENV=b" ...
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
i=0
for envs in "$@"; do
  i=$((i+1))
  env $envs timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab_$i.log 2>&1
  echo "== $envs"; tail -1 gpurun_out/ab_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stages_ms'], d['e2e']['ms_per_step'], d['roofline']['avg_launch_ms'], d.get('roofline_scatter'))"
done
timeout 600 python tools/timeline.py > gpurun_out/timeline.txt 2>&1; head -40 gpurun_out/timeline.txt
