#!/bin/bash
# Bench lines for the other configurations / modes.  usage: tools/gpu_configs.sh TAG
TAG=${1:-c}
mkdir -p gpurun_out
for args in "--config 2 --argmax 2" "--config 1" "--config 4 --steps 5 --warmup 3"; do
  name=$(echo $args | tr -d ' -')
  timeout 900 python bench.py --no-cpu-baseline $args > gpurun_out/${TAG}_${name}.json 2> gpurun_out/${TAG}_${name}.err
  python -c "
import json
d=json.load(open('gpurun_out/${TAG}_${name}.json'))
print('$args', 'value %.4g'%d['value'], 'ms %.4f'%d['ms_per_step'], 'e2e %.4g'%d['e2e']['value'], 'qevals/s %.3g'%d['q_evals_per_s'])
print({k:round(v,4) for k,v in d['kernels_ms_per_step'].items()})
" || tail -5 gpurun_out/${TAG}_${name}.err
done
