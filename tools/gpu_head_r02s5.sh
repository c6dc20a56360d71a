# HEAD check of the last round-2 session: GPU suite, smoke, bench (headline + reference arm).
#   gpurun --timeout 1800 -- 'bash tools/gpu_head_r02s5.sh'
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02s5_gputest.log 2>&1; echo "gpu tests rc=$?" >> gpurun_out/r02s5_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02s5_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02s5_smoke.log
timeout 900 python bench.py > gpurun_out/r02s5_bench.json 2> gpurun_out/r02s5_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r02s5_bench_reference_arm.json 2> gpurun_out/r02s5_bench_ref.err
