# BASELINE configs beyond C2 on one B200: C4 (Qwen2.5-VL-7B LM, 24 x 1280 image chunks + text),
# C3 at 1 GPU (128K ctx, info-flow reorder), C5 recompute-ratio sweep at 32K and 128K.
mkdir -p gpurun_out/configs_r2
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
run() { name=$1; shift; timeout 900 python bench.py --no-cpu-baseline --steps 3 --warmup 3 "$@" > gpurun_out/configs_r2/$name.log 2>&1; tail -1 gpurun_out/configs_r2/$name.log | cut -c1-300; }
run c4 --model qwen25vl_7b
run c2_reorder --reorder
for r in 0.05 0.10 0.20 0.30; do run c5_32k_r$r --ratio $r; done
run c3_128k_reorder --ctx 131072 --reorder
for r in 0.05 0.15 0.30; do run c5_128k_r$r --ctx 131072 --ratio $r; done
