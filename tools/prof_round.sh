# Round profiling recipe (run under gpurun): bench line (VGG-16 b256 headline),
# the other BASELINE configs, launch list of one dyn step with DRAM bytes,
# per-layer times, and full ncu captures of the top conv kernels.
set -x
LABEL=${LABEL:-r01s3}
timeout 600 python bench.py > gpurun_out/bench_${LABEL}.json 2> gpurun_out/bench_${LABEL}.err
for net in alexnet overfeat inception_toy; do
  timeout 300 python bench.py --net $net --batch 128 --policies dyn,all,conv,none --no-cpu-baseline > gpurun_out/bench_$net.json 2> gpurun_out/bench_$net.err
done
timeout 1200 python bench.py --extra 400 --batch 32 --policies dyn,dynt,none --steps 2 --no-cpu-baseline > gpurun_out/bench_vgg416.json 2> gpurun_out/bench_vgg416.err
python tools/prof_layers.py vgg16 256 none > gpurun_out/layers_none.txt 2>&1
python tools/prof_layers.py alexnet 128 none > gpurun_out/layers_alexnet.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${LABEL}_launches_dyn.csv python bench.py --policies dyn --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"tc_conv_pair|tc_wgrad_pair|tc_conv_halo|tc_wgrad_halo|c3tc" --launch-skip 0 --launch-count 7 -o gpurun_out/${LABEL}_full python tools/one_step.py vgg16 256 none > gpurun_out/ncu_full.log 2>&1
# backward-pass kernels (one launch each): pair wgrad, pair-halo wgrad, first-layer wgrad, persistent FC wgrad, pool bwd
ncu --set full --clock-control none --import-source on -k regex:"tc_wgrad_pair|tc_wgrad_halo_pair|c3tc_wgrad|tc_conv_persist|maxpool2x2_bwd" --launch-skip 0 --launch-count 12 -o gpurun_out/${LABEL}_full_bwd python tools/one_step.py vgg16 256 none > gpurun_out/ncu_full_bwd.log 2>&1
ls -la gpurun_out
