mkdir -p gpurun_out
timeout 300 python tools/attn_bench.py ${ATTN_LIBS} > gpurun_out/attn_ab.txt 2>&1
[ -n "$TRACE_LIB" ] && python tools/attn_trace.py $TRACE_LIB > gpurun_out/attn_trace.txt 2>&1
[ -n "$SCATTER_LIBS" ] && python tools/scatter_bench.py $SCATTER_LIBS > gpurun_out/scatter_ab.txt 2>&1
cat gpurun_out/attn_ab.txt gpurun_out/attn_trace.txt gpurun_out/scatter_ab.txt
