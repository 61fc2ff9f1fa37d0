# compute-sanitizer passes over tools/sanitize_run.py (logs under gpurun_out/)
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 $CS --tool $tool --print-limit 50 python tools/sanitize_run.py > gpurun_out/r2_sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/r2_sanitizer_summary.txt
  tail -3 gpurun_out/r2_sanitizer_$tool.txt >> gpurun_out/r2_sanitizer_summary.txt
done
cat gpurun_out/r2_sanitizer_summary.txt
