mkdir -p gpurun_out/r02s4_configs
for cfg in "alexnet 128 0 all,allb,none,noneb" "overfeat 128 0 conv,convb,none,noneb" "inception_toy 128 0 dyn,dynb,none,noneb" "vgg16 32 400 dyn,dynb,dynz,dynzb"; do
  set -- $cfg
  timeout 900 python bench.py --net $1 --batch $2 --extra $3 --policies $4 --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/r02s4_configs/$1_b$2_e$3.json 2> gpurun_out/r02s4_configs/$1_b$2_e$3.err
  echo "$1 b$2 e$3 rc=$?"
  python -c "
import json,sys; d=json.load(open('gpurun_out/r02s4_configs/$1_b$2_e$3.json'))
for k,v in d['policies'].items(): print('  ',k, v.get('label'), v.get('verdict'), v.get('images_per_s'), v.get('ms_per_step'), v.get('offload_bytes_per_iter'), v.get('conv_fc_tflops'))
"
done
