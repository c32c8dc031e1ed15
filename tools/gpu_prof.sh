# One GPU call: timeline of a warm step, ncu launch list, ncu --set full of the main kernels.
# NCU_KERNELS entries are name:regex:skip (skip = matching launches to pass over first).
set -x
mkdir -p gpurun_out/ncu
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python tools/timeline.py > gpurun_out/timeline.txt 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/ncu/launches.csv python bench.py --ncu --warmup 1 > /dev/null 2>&1
DEFAULT="recompute_attn_tc:recompute_attn_v5:1 rotate_rows:rotate_rows:0 qkv_rope_scatter:qkv_rope_scatter_bf16:1 add_rmsnorm:add_rmsnorm_pf:1 silu_mul:silu_mul_bf16_fast:1 prompt_attn_tc:prompt_attn_tc:1 assemble_gather:assemble_gather:0 prompt_mm:prompt_mm_kernel:2"
for spec in ${NCU_KERNELS:-$DEFAULT}; do
  IFS=: read name rx skip <<< "$spec"
  timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:$rx -s $skip -c 1 \
    -o gpurun_out/ncu/$name -f python bench.py --ncu --warmup 1 > gpurun_out/ncu/$name.log 2>&1
done
python tools/ncu_traffic.py gpurun_out/ncu/*.ncu-rep > gpurun_out/ncu/traffic.json
ls -la gpurun_out/ncu
