# prompt_mm ring depth A/B (select stage of the C2 step), 2 rounds
mkdir -p gpurun_out/pmm_ab
for r in 1 2; do
for spec in cur:paper_2603_05353_b200/_build/libifkv.so:2 s8:_ab/s8/libifkv.so:1 s2:_ab/s2/libifkv.so:3 s2b:_ab/s2/libifkv.so:4; do
  IFS=: read name lib psm <<< "$spec"
  IFKV_LIB=$lib IFKV_PMM_PER_SM=$psm timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sdpa-comparator > gpurun_out/pmm_ab/$name.$r.log 2>&1
  echo "$name r$r $(tail -1 gpurun_out/pmm_ab/$name.$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), {k: round(v,3) for k,v in d["stages_ms"].items()}, "pmm", round(d["roofline_prompt_mm"]["ms_all_layers"],3), d["clocks"]["sm_mhz"])')"
done; done
