# Dh=128 SIMT prompt partial: parity tests, C2 / C3 steps, one first-pass launch under ncu
timeout 900 python -m pytest tests/test_gpu_path.py tests/test_gpu_kernels.py -x -q -m gpu > gpurun_out/pd128_tests.log 2>&1; tail -2 gpurun_out/pd128_tests.log
timeout 900 python -m pytest tests/test_gpu_headline.py -x -q -m gpu > gpurun_out/pd128_headline.log 2>&1; tail -2 gpurun_out/pd128_headline.log
for r in 1 2; do for a in "" "--reorder"; do
timeout 600 python bench.py $a --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-sdpa-comparator > gpurun_out/pd128_bench$a.$r.log 2>&1
tail -1 gpurun_out/pd128_bench$a.$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("'$a'", round(d["ms_per_step"],2), {k: round(x,2) for k,x in d["stages_ms"].items()}, d["clocks"]["sm_mhz"])'
done; done
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"prompt_attn_partial" --launch-skip 3 --launch-count 2 --csv python tools/timeline.py --reorder --out gpurun_out/tl_tmp.json 2>/dev/null | grep -E "prompt_attn_partial" | cut -c1-60,250-400 > gpurun_out/pd128_ncu.txt; cat gpurun_out/pd128_ncu.txt
