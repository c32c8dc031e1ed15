# v10 default = early P halves + 25 % FMA-pipe exp2: tests, in-step A/B vs the
# plain v10, bench lines, ncu of the attention kernel
set -x
mkdir -p gpurun_out/ncu
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -rf -s > gpurun_out/pytest_gpu3.log 2>&1; echo pytest=$?
grep -E "passed|failed" gpurun_out/pytest_gpu3.log | tail -2; grep "selection: k=" gpurun_out/pytest_gpu3.log
bash tools/gpu_ab_libs.sh v10plain=_ab/v10ns/libifkv.so v10new=paper_2603_05353_b200/_build/libifkv.so
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:recompute_attn_v10 -s 1 -c 1 \
  -o gpurun_out/ncu/recompute_attn_tc -f python bench.py --ncu --warmup 1 > gpurun_out/ncu/recompute_attn_tc.log 2>&1; echo ncu=$?
python tools/ncu_traffic.py gpurun_out/ncu/recompute_attn_tc.ncu-rep > gpurun_out/ncu/traffic_attn.json 2>&1
tail -1 gpurun_out/bench.log | cut -c1-300
