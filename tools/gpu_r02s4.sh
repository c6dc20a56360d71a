mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_bf16_gpu.py -x -q > gpurun_out/r02s4_bf16_tests.log 2>&1
echo "bf16 tests rc=$?" >> gpurun_out/r02s4_bf16_tests.log
timeout 300 python tools/prof_layers.py vgg16 256 none --bf16 > gpurun_out/r02s4_layers_bf16_pad.txt 2>&1
VDNN_BF16_PAD=0 timeout 300 python tools/prof_layers.py vgg16 256 none --bf16 > gpurun_out/r02s4_layers_bf16_nopad.txt 2>&1
tail -3 gpurun_out/r02s4_bf16_tests.log; head -3 gpurun_out/r02s4_layers_bf16_pad.txt; tail -1 gpurun_out/r02s4_layers_bf16_pad.txt; head -3 gpurun_out/r02s4_layers_bf16_nopad.txt; tail -1 gpurun_out/r02s4_layers_bf16_nopad.txt
