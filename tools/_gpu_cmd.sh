mkdir -p gpurun_out/sanitizer; bash tools/sanitize.sh > gpurun_out/sanitizer/summary.txt 2>&1
