mkdir -p gpurun_out
timeout 600 python bench.py --policies dyn,dynb,none,noneb --no-cpu-baseline --artifacts gpurun_out/r02_artifacts > gpurun_out/r02s3_bench_b.json 2> gpurun_out/r02s3_bench_b.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02s3_launches_dyn.csv python tools/one_step.py vgg16 256 dyn > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02s3_launches_dynb.csv python tools/one_step.py vgg16 256 dyn --bf16 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"tcb_conv" --launch-skip 6 --launch-count 4 -o gpurun_out/r02s3_full_bf16 python tools/one_step.py vgg16 256 none --bf16 > gpurun_out/ncu_full_bf16.log 2>&1
ls -la gpurun_out | tail -20
