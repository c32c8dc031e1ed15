# prompt_qkv early exit: reorder / selection parity + C3 timeline + C2/C3 bench
timeout 900 python -m pytest tests/test_gpu_path.py tests/test_gpu_kernels.py -x -q -m gpu > gpurun_out/c3qkv_tests.log 2>&1; tail -2 gpurun_out/c3qkv_tests.log
timeout 900 python -m pytest tests/test_gpu_headline.py -x -q -m gpu > gpurun_out/c3qkv_headline.log 2>&1; tail -2 gpurun_out/c3qkv_headline.log
timeout 600 python tools/timeline.py --reorder --out gpurun_out/timeline_c3b.json > gpurun_out/timeline_c3b.txt 2>&1; grep -E "span|prompt_qkv|prompt_attn_merge" gpurun_out/timeline_c3b.txt | head -4
for a in "" "--reorder"; do
timeout 600 python bench.py $a --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-sdpa-comparator > gpurun_out/c3qkv_bench$a.log 2>&1
tail -1 gpurun_out/c3qkv_bench$a.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("'$a'", round(d["ms_per_step"],2), d["stages_ms"], d["clocks"]["sm_mhz"])'
done
