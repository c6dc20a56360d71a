mkdir -p gpurun_out/r02s4_sanitizer
for t in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_step.py > gpurun_out/r02s4_sanitizer/$t.log 2>&1
  echo "$t rc=$?"; tail -n 3 gpurun_out/r02s4_sanitizer/$t.log
done
