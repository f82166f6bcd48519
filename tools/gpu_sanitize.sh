# compute-sanitizer over tools/sanitize_paths.py: memcheck, racecheck, synccheck, initcheck
set -x
O=gpurun_out/r02/sanitizer; mkdir -p $O
timeout 600 python tools/sanitize_paths.py > $O/plain.log 2>&1; echo "plain rc=$?"; tail -2 $O/plain.log
for tool in ${TOOLS:-memcheck synccheck initcheck}; do
  timeout 1800 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit ${PRINT_LIMIT:-50} python tools/sanitize_paths.py > $O/$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 $O/$tool.log
done
