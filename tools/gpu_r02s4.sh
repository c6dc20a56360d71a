mkdir -p gpurun_out
START=$(date +%s)
timeout 1200 python bench.py --artifacts gpurun_out/r02s4_artifacts_final > gpurun_out/r02s4_bench_final.json 2> gpurun_out/r02s4_bench_final.err
echo "bench rc=$? wall=$(( $(date +%s) - START ))s"
START=$(date +%s)
timeout 900 python bench.py --impl reference > gpurun_out/r02s4_bench_ref_final.json 2> gpurun_out/r02s4_bench_ref_final.err
echo "ref rc=$? wall=$(( $(date +%s) - START ))s"
for cfg in "alexnet 128 0 all,allb,none,noneb" "overfeat 128 0 conv,convb,none,noneb"; do
  set -- $cfg
  timeout 900 python bench.py --net $1 --batch $2 --extra $3 --policies $4 --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r02s4_configs/$1_b$2_e$3.json 2> gpurun_out/r02s4_configs/$1_b$2_e$3.err
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02s4_launches_dyn_final.csv python tools/one_step.py vgg16 256 dyn > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02s4_launches_noneb_final.csv python tools/one_step.py vgg16 256 none --bf16 > /dev/null 2>&1
