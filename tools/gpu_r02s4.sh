mkdir -p gpurun_out
timeout 300 python tools/prof_layers.py vgg16 256 none --precise > gpurun_out/r02s4_layers_precise.txt 2>&1
cat gpurun_out/r02s4_layers_precise.txt | awk '$2=="conv"||$2=="fc"||$2=="pool"||$2=="total"'
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02s4_launches_nonef.csv python tools/one_step.py vgg16 64 none > /dev/null 2>&1
