# One GPU call: timeline of a warm step, ncu launch list, ncu --set full of the main kernels.
set -x
mkdir -p gpurun_out/ncu
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python tools/timeline.py > gpurun_out/timeline.txt 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/ncu/launches.csv python bench.py --ncu --warmup 1 > /dev/null 2>&1
for k in ${NCU_KERNELS:-rotate_rows qkv_rope_scatter_vec silu_mul_bf16x8 add_rmsnorm_kernel recompute_attn_tc prompt_attn_tc assemble_gather}; do
  timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:$k -c 1 \
    -o gpurun_out/ncu/$k -f python bench.py --ncu --warmup 1 > gpurun_out/ncu/$k.log 2>&1
done
ls -la gpurun_out/ncu
