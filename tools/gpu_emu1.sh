# attention with 12.5 % FMA-pipe exponentials: GPU tests + bench
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/emu1_pytest.log 2>&1; tail -1 gpurun_out/emu1_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/emu1_smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > gpurun_out/emu1_bench.log 2>&1; tail -1 gpurun_out/emu1_bench.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), d["stages_ms"], d["roofline"]["frac"], d["roofline"]["avg_launch_ms"], d["clocks"]["sm_mhz"], d["e2e"]["ms_per_step"])'
