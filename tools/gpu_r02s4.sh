mkdir -p gpurun_out
timeout 300 python tools/prof_layers.py vgg16 256 none --bf16 > gpurun_out/r02s4_layers_bf16_pair2.txt 2>&1
awk '$2=="conv"||$2=="fc"||$2=="pool"' gpurun_out/r02s4_layers_bf16_pair2.txt; tail -1 gpurun_out/r02s4_layers_bf16_pair2.txt
timeout 900 python -m pytest tests/test_bf16_gpu.py -x -q > gpurun_out/r02s4_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02s4_tests.log
tail -n 30 gpurun_out/r02s4_tests.log
