# compute-sanitizer over tools/sanitize_cases.py (one tool at a time); logs to gpurun_out/
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report all"
  [ $tool = memcheck ] && extra="--leak-check no"
  timeout ${SAN_TIMEOUT:-1500} $CS --tool $tool $extra --print-limit 50 python tools/sanitize_cases.py ${CASES:-} \
    > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|ok$' gpurun_out/sanitize_$tool.log | tr '\n' ' ')"
done
