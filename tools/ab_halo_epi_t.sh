# A/B of the TF32 halo-pair transposed-store epilogue (store_half32_f32; VDNN_HALO_EPI_T=0 = per-lane row stores).
#   gpurun --timeout 1800 -- 'bash tools/ab_halo_epi_t.sh'
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_layer_parity_gpu.py -m gpu -x -q > gpurun_out/r02s5c_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02s5c_tests.log
for r in 1 2; do
  for t in 0 1; do
    VDNN_HALO_EPI_T=$t timeout 300 python tools/prof_layers.py vgg16 256 none > gpurun_out/r02s5c_layers_tf32_epit$t.r$r.txt 2>&1
  done
done
for t in 0 1; do
  VDNN_HALO_EPI_T=$t timeout 600 python bench.py --policies none --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/r02s5c_bench_none_epit$t.json 2>&1
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__throughput.avg.pct_of_peak_sustained_active --clock-control none --csv \
  -k regex:"tc_conv_halo_pair_kernel" --launch-count 8 --log-file gpurun_out/r02s5c_ncu_halo_pair_epit1.csv python tools/one_step.py vgg16 256 none > /dev/null 2>&1
