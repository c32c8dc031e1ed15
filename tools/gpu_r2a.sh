mkdir -p gpurun_out/ncu
bash tools/gpu_round.sh > gpurun_out/round.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/ncu/launches.csv python bench.py --ncu --warmup 1 > gpurun_out/ncu/launches.log 2>&1
echo launches=$?
