mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_path.py -x -q -k "query_graph or store_path" > gpurun_out/pytest_graph.log 2>&1; echo pytest=$?; tail -15 gpurun_out/pytest_graph.log
timeout 900 python bench.py --no-cpu-baseline --no-sdpa-comparator > gpurun_out/bench_graph.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_graph.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['eager_ms_per_step'], d['e2e']['ms_per_step'], d['gpu_launches'], d['stages_ms'], d['clocks'])"
tail -5 gpurun_out/bench_graph.log | cut -c1-400
