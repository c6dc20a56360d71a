mkdir -p gpurun_out
timeout 600 python tools/algo_probe.py 32 > gpurun_out/r02s4_algo_probe.txt 2>&1
cat gpurun_out/r02s4_algo_probe.txt
