mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"c3" --csv --log-file gpurun_out/r02s4_launches_c3_v2.csv python tools/one_step.py vgg16 256 none > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"c3" --csv --log-file gpurun_out/r02s4_launches_c3b_v2.csv python tools/one_step.py vgg16 256 none --bf16 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_bf16_gpu.py tests/test_layer_parity_gpu.py -x -q 2>&1 | tail -n 2
