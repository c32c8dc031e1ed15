# mufu throughput micro-benchmark + ncu --set full of the main kernels of the current step
set -x
mkdir -p gpurun_out/ncu gpurun_out/micro
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mufu_bench tools/micro/mufu_bench.cu && /tmp/mufu_bench > gpurun_out/micro/mufu.txt 2>&1
cat gpurun_out/micro/mufu.txt
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for spec in recompute_attn_tc:recompute_attn_v5:1 gemm_pair_qkv:gemm_pair_kernel:4 gemm_pair_swiglu:gemm_pair_kernel:6 prompt_attn_tc:prompt_attn_tc:1 assemble_gather:assemble_gather:0 prompt_mm:prompt_mm_kernel:2; do
  IFS=: read name rx skip <<< "$spec"
  timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:$rx -s $skip -c 1 \
    -o gpurun_out/ncu/$name -f python bench.py --ncu --warmup 1 > gpurun_out/ncu/$name.log 2>&1
done
python tools/ncu_traffic.py gpurun_out/ncu/*.ncu-rep > gpurun_out/ncu/traffic.json
cat gpurun_out/ncu/traffic.json
