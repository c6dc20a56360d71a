# Final evidence of the last round-2 session (HEAD with the transposed-store epilogues):
#   gpurun --timeout 3600 -- 'bash tools/gpu_final_r02s5.sh'
set -u
mkdir -p gpurun_out/r02s5_sanitizer
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02s5f_gputest.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/r02s5f_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02s5f_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02s5f_smoke.log
timeout 900 python bench.py > gpurun_out/r02s5f_bench.json 2> gpurun_out/r02s5f_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r02s5f_bench_reference_arm.json 2> gpurun_out/r02s5f_bench_ref.err
for pol in "dyn" "none" "none --bf16"; do
  tag=$(echo "$pol" | tr -d ' -')
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/r02s5f_launches_$tag.csv python tools/one_step.py vgg16 256 $pol > /dev/null 2>&1
done
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_step.py > gpurun_out/r02s5_sanitizer/$t.log 2>&1
  echo "rc=$?" >> gpurun_out/r02s5_sanitizer/$t.log
done
