# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_driver.py;
# one summary line per tool into gpurun_out/sanitize_summary.txt
mkdir -p gpurun_out
: > gpurun_out/sanitize_summary.txt
for tool in memcheck racecheck synccheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 --log-file gpurun_out/sanitize_$tool.log \
      python tools/sanitize_driver.py > gpurun_out/sanitize_${tool}_stdout.log 2>&1
  rc=$?
  echo "$tool rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/sanitize_$tool.log | tail -3 | tr '\n' ' ')" >> gpurun_out/sanitize_summary.txt
done
