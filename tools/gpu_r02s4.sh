mkdir -p gpurun_out
REPS=2 timeout 300 python tools/bench_conv.py precise
timeout 600 python -m pytest tests/test_kernels_gpu.py -x -q 2>&1 | tail -n 2
