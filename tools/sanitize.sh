# compute-sanitizer memcheck / racecheck / synccheck on small caches (HBM and
# half offloaded), every product mode, diag, export, PCG, LM direction
mkdir -p gpurun_out/sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_workload.py 20 > gpurun_out/sanitizer/$tool.log 2>&1
  echo "$tool rc=$? $(tail -1 gpurun_out/sanitizer/$tool.log)"
done
