#!/bin/bash
# A/B of the split-K count of the weight-gradient GEMMs (HRP_WGRAD_DIV).  usage: tools/gpu_wgrad_ab.sh TAG
TAG=${1:-w}
mkdir -p gpurun_out
for rep in 1 2; do
  for div in 1 2 3 4; do
    for args in "--config 2" "--config 4 --steps 5 --warmup 3"; do
      name=$(echo $args | tr -d ' -')_div${div}_${rep}
      HRP_WGRAD_DIV=$div timeout 600 python bench.py --no-cpu-baseline $args > gpurun_out/${TAG}_${name}.json 2> gpurun_out/${TAG}_${name}.err
      python -c "
import json
d=json.load(open('gpurun_out/${TAG}_${name}.json'))
print('$name', 'ms %.4f'%d['ms_per_step'], {k:round(v,4) for k,v in d['kernels_ms_per_step'].items() if k in ('gemm_bwd','misc')})
" || tail -3 gpurun_out/${TAG}_${name}.err
    done
  done
done
