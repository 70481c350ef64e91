# compute-sanitizer memcheck / racecheck / synccheck on a small cache + products
mkdir -p gpurun_out/sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/dbg_stream.py 20 > gpurun_out/sanitizer/$tool.log 2>&1
  echo "$tool rc=$? $(grep -c 'ERROR SUMMARY: 0 errors\|RACECHECK SUMMARY: 0 hazards' gpurun_out/sanitizer/$tool.log) $(tail -1 gpurun_out/sanitizer/$tool.log)"
done
