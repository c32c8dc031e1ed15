# rotating-gather CTAs per SM (IFKV_GATHER_CPS), C2 assemble stage, 2 rounds
mkdir -p gpurun_out/cps_ab
for r in 1 2; do for c in 8 4 16 32; do
  IFKV_GATHER_CPS=$c timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sdpa-comparator > gpurun_out/cps_ab/$c.$r.log 2>&1
  echo "cps$c r$r $(tail -1 gpurun_out/cps_ab/$c.$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), {k: round(v,3) for k,v in d["stages_ms"].items()}, d["clocks"]["sm_mhz"])')"
done; done
