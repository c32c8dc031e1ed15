# scorer work-item length A/B (IFKV_PROMPT_ITEM_KEYS), C2 select stage, 2 rounds
mkdir -p gpurun_out/ik_ab
for r in 1 2; do for ik in default 1536 1792 1280 1024; do
  if [ $ik = default ]; then unset IFKV_PROMPT_ITEM_KEYS; else export IFKV_PROMPT_ITEM_KEYS=$ik; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sdpa-comparator > gpurun_out/ik_ab/$ik.$r.log 2>&1
  echo "$ik r$r $(tail -1 gpurun_out/ik_ab/$ik.$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), {k: round(v,3) for k,v in d["stages_ms"].items()}, d["selection_parity"]["swapped_pairs_vs_fp64_scoring"] if d.get("selection_parity") else None, d["clocks"]["sm_mhz"])')"
done; done
