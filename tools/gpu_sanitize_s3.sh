mkdir -p gpurun_out/san
for t in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_c1.py > gpurun_out/san/$t.log 2>&1; echo "$t rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error" gpurun_out/san/$t.log | sort | uniq -c | head -5
done
