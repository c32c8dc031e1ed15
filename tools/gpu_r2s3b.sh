# session-3 round check with the v10 attention default: smoke, GPU tests,
# bench (ours + reference arm), launch list, ncu --set full of the main
# kernels, compute-sanitizer on the C1 pass.
set -x
mkdir -p gpurun_out/ncu gpurun_out/san
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo ref=$?
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/ncu/launches.csv python bench.py --ncu --warmup 1 > /dev/null 2>&1; echo launches=$?
for spec in recompute_attn_tc:recompute_attn_v10:1 gemm_pair:gemm_pair_kernel:1 assemble_gather:assemble_gather_rotate:0 prompt_attn_tc:prompt_attn_tc:1 prompt_mm:prompt_mm_kernel:2 add_rmsnorm:add_rmsnorm_pf:1; do
  IFS=: read name rx skip <<< "$spec"
  timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:$rx -s $skip -c 1 \
    -o gpurun_out/ncu/$name -f python bench.py --ncu --warmup 1 > gpurun_out/ncu/$name.log 2>&1; echo ncu_$name=$?
done
python tools/ncu_traffic.py gpurun_out/ncu/*.ncu-rep > gpurun_out/ncu/traffic.json 2>gpurun_out/ncu/traffic.err
for t in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $t python tools/sanitize_c1.py > gpurun_out/san/$t.log 2>&1; echo san_$t=$?
  tail -2 gpurun_out/san/$t.log
done
tail -1 gpurun_out/bench.log | cut -c1-600
