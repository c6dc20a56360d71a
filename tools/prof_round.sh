set -x
python tools/prof_layers.py vgg16 256 none > gpurun_out/layers_none.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r01s2_launches_dyn.csv python bench.py --policies dyn --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc_conv --launch-skip 2 --launch-count 4 -o gpurun_out/r01s2_conv_full python tools/one_step.py vgg16 256 none > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
