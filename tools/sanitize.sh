# compute-sanitizer over every library entry point (tools/sanitize_run.py),
# our kernels only (namespace lseg); logs in gpurun_out/sanitize_<tool>.log
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 300 python tools/sanitize_run.py > gpurun_out/sanitize_plain.log 2>&1; echo plain rc=$?
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check no"
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  timeout ${SAN_TIMEOUT:-1500} $CS --tool $tool $extra --kernel-name regex:lseg --error-exitcode 7 \
      --print-limit 50 python tools/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo $tool rc=$?; grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|all ok' gpurun_out/sanitize_$tool.log | tail -3
done
