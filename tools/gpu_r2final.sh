# final round-2 capture with the default library: smoke, GPU tests, bench +
# reference arm, launch list of one step, ncu --set full of the attention
set -x
mkdir -p gpurun_out/final
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -rf -s > gpurun_out/final/pytest_gpu.log 2>&1; echo pytest=$?
grep -E "passed|failed" gpurun_out/final/pytest_gpu.log | tail -1
timeout 600 python bench.py > gpurun_out/final/bench.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference > gpurun_out/final/bench_ref.log 2>&1; echo ref=$?
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/final/launches.csv python bench.py --ncu --warmup 1 > /dev/null 2>&1; echo launches=$?
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:recompute_attn_v10 -s 1 -c 1 \
  -o gpurun_out/final/recompute_attn_tc -f python bench.py --ncu --warmup 1 > gpurun_out/final/ncu_attn.log 2>&1; echo ncu=$?
python tools/ncu_traffic.py gpurun_out/final/recompute_attn_tc.ncu-rep > gpurun_out/final/traffic_attn.json 2>&1
python tools/ncu_stalls.py gpurun_out/final/recompute_attn_tc.ncu-rep 12 > gpurun_out/final/ncu_attn_stalls.txt 2>&1
rm -f gpurun_out/final/recompute_attn_tc.ncu-rep
tail -1 gpurun_out/final/bench.log | cut -c1-300
