mkdir -p gpurun_out
timeout 300 python tools/prof_layers.py vgg16 256 none --bf16 > gpurun_out/r02s4_layers_bf16_v6.txt 2>&1
awk '$2=="conv"||$2=="fc"' gpurun_out/r02s4_layers_bf16_v6.txt | tail -13; tail -1 gpurun_out/r02s4_layers_bf16_v6.txt
timeout 300 python tools/prof_layers.py alexnet 128 none --bf16 > gpurun_out/r02s4_layers_alexnet_bf16.txt 2>&1
awk '$2=="fc"||$2=="total"' gpurun_out/r02s4_layers_alexnet_bf16.txt
timeout 900 python -m pytest tests/test_bf16_gpu.py -x -q 2>&1 | tail -n 2
