# A/B of the BF16 transposed-store epilogue (store_tile32_t; VDNN_BF16_EPI_T=0 is the old per-lane store).
#   gpurun --timeout 1800 -- 'bash tools/ab_epi_t.sh'
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_bf16_gpu.py -m gpu -x -q > gpurun_out/r02s5b_epit_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02s5b_epit_tests.log
for r in 1 2; do
  for t in 0 1; do
    VDNN_BF16_EPI_T=$t timeout 300 python tools/prof_layers.py vgg16 256 none --bf16 > gpurun_out/r02s5b_layers_bf16_epit$t.r$r.txt 2>&1
  done
done
for t in 0 1; do
  VDNN_BF16_EPI_T=$t timeout 600 python bench.py --policies noneb,dynzb --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/r02s5b_bench_bf16_epit$t.json 2>&1
done
