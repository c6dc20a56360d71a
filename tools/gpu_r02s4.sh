mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --kernel-name-base demangled -k regex:"halo" --csv --log-file gpurun_out/r02s4_launches_haloB.csv python tools/one_step.py vgg16 256 none --bf16 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_layer_parity_gpu.py tests/test_bf16_gpu.py -x -q 2>&1 | tail -n 2
