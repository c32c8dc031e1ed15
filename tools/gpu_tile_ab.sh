# GEMM tile width A/B (IFKV_GEMM_TILE=1000+BN for every GEMM), C2 step, 2 rounds
mkdir -p gpurun_out/tile_ab
for r in 1 2; do for t in 0 1256; do
  IFKV_GEMM_TILE=$t timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-sdpa-comparator > gpurun_out/tile_ab/$t.$r.log 2>&1
  echo "tile$t r$r $(tail -1 gpurun_out/tile_ab/$t.$r.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],2), {k: round(v,3) for k,v in d["stages_ms"].items()}, round(d["roofline_gemm"]["ms_per_step"],2), d["clocks"]["sm_mhz"])')"
done; done
