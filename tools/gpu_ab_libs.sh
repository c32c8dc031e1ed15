# Interleaved in-step A/B of library variants: bash tools/gpu_ab_libs.sh name=path/libifkv.so ... (2 rounds)
mkdir -p gpurun_out/ab
for r in 1 2; do
  for spec in "$@"; do
    name=${spec%%=*}; lib=${spec#*=}
    IFKV_LIB=$lib timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sdpa-comparator > gpurun_out/ab/$name.$r.log 2>&1
    echo "$name r$r $(tail -1 gpurun_out/ab/$name.$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), {k: round(v,2) for k,v in d["stages_ms"].items()}, "attn", round(d["roofline"]["avg_launch_ms"],3), "clk", d["clocks"]["sm_mhz"])')"
  done
done
