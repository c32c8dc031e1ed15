# In-step A/B of programmatic dependent launch in the scoring pass (IFKV_PDL)
mkdir -p gpurun_out/ab
for r in 1 2; do
  for v in 0 1; do
    IFKV_PDL=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sdpa-comparator > gpurun_out/ab/pdl$v.$r.log 2>&1
    echo "pdl=$v r$r $(tail -1 gpurun_out/ab/pdl$v.$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), {k: round(v,2) for k,v in d["stages_ms"].items()}, "pmm", round(d["roofline_prompt_mm"]["ms_all_layers"],3), "clk", d["clocks"]["sm_mhz"])')"
  done
done
