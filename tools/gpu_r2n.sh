python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -2
for lib in _ab/gold/libifkv.so paper_2603_05353_b200/_build/libifkv.so; do echo "== $lib"; IFKV_LIB=$lib timeout 600 python tools/prefill_prof.py 2>&1 | grep -E "==|gemm_pair|recompute_attn" ; done
bash tools/gpu_ab_libs.sh old=_ab/gold/libifkv.so band=paper_2603_05353_b200/_build/libifkv.so
