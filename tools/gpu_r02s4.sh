mkdir -p gpurun_out
timeout 300 python tools/prof_layers.py alexnet 128 none --bf16 > gpurun_out/r02s4_layers_alexnet_bf16.txt 2>&1
timeout 300 python tools/prof_layers.py overfeat 128 none --bf16 > gpurun_out/r02s4_layers_overfeat_bf16.txt 2>&1
head -1 gpurun_out/r02s4_layers_alexnet_bf16.txt; tail -1 gpurun_out/r02s4_layers_alexnet_bf16.txt; head -1 gpurun_out/r02s4_layers_overfeat_bf16.txt; tail -1 gpurun_out/r02s4_layers_overfeat_bf16.txt
timeout 1200 python -m pytest tests/test_bf16_gpu.py -x -q -k "alexnet or overfeat or vocab or json" 2>&1 | tail -n 3
