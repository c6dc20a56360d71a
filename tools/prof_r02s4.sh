# Evidence recipe of the round-2 HEAD (run on one B200 through gpurun, from the repo root):
#   gpurun --timeout 3600 -- 'bash tools/prof_r02s4.sh'
# Outputs land in gpurun_out/; the committed copies are under profiles/r02s4_*.
set -u
mkdir -p gpurun_out/r02s4_configs gpurun_out/r02s4_sanitizer
# bench lines (headline + reference arm), measured artefacts of the dyn / dynb steps
timeout 1200 python bench.py --artifacts gpurun_out/r02s4_artifacts > gpurun_out/r02s4_bench.json 2> gpurun_out/r02s4_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r02s4_bench_reference_arm.json 2> gpurun_out/r02s4_bench_ref.err
# the other BASELINE configs, fp32 and BF16 storage
for cfg in "alexnet 128 0 all,allb,none,noneb" "overfeat 128 0 conv,convb,none,noneb" \
           "inception_toy 128 0 dyn,dynb,none,noneb" "vgg16 32 400 dyn,dynb,dynz,dynzb"; do
  set -- $cfg
  timeout 900 python bench.py --net $1 --batch $2 --extra $3 --policies $4 --no-cpu-baseline --steps 5 --warmup 3 \
    > gpurun_out/r02s4_configs/$1_b$2_e$3.json 2> gpurun_out/r02s4_configs/$1_b$2_e$3.err
done
# per-layer times
python tools/prof_layers.py vgg16 256 none --bf16 > gpurun_out/r02s4_layers_vgg16_b256_none_bf16.txt 2>&1
python tools/prof_layers.py vgg16 256 none > gpurun_out/r02s4_layers_vgg16_b256_none_tf32.txt 2>&1
python tools/prof_layers.py alexnet 128 none --bf16 > gpurun_out/r02s4_layers_alexnet_b128_none_bf16.txt 2>&1
python tools/prof_layers.py overfeat 128 none --bf16 > gpurun_out/r02s4_layers_overfeat_b128_none_bf16.txt 2>&1
python tools/algo_probe.py 32 > gpurun_out/r02s4_algo_probe.txt 2>&1
# ncu launch lists (per-kernel share of one step; summarize with tools/summarize_launches.py --steps 2)
for pol in "dyn" "dyn --bf16" "none --bf16"; do
  tag=$(echo "$pol" | tr -d ' -')
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/r02s4_launches_$tag.csv python tools/one_step.py vgg16 256 $pol > /dev/null 2>&1
done
# full captures of the BF16 kernels
ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"tcb_pair_kernel|tcb_halo_kernel|tcb_wgrad_halo_kernel|c3b_fprop|c3b_wgrad_kernel|maxpool2x2_bwd_b|maxpool2x2_fwd_b" \
  --launch-count 12 -o gpurun_out/r02s4_full_bf16 python tools/one_step.py vgg16 256 none --bf16 > gpurun_out/ncu_full_bf16.log 2>&1
# compute-sanitizer over every kernel family
for t in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_step.py > gpurun_out/r02s4_sanitizer/$t.log 2>&1
done
