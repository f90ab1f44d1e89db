#!/bin/bash
# Bench lines of every configuration (round 2).  usage: tools/gpu_final_r2.sh TAG
TAG=${1:-r2q}
mkdir -p gpurun_out
run() {
  name=$1; shift
  timeout 900 python bench.py "$@" > gpurun_out/${TAG}_${name}.json 2> gpurun_out/${TAG}_${name}.err
  python -c "
import json
d=json.load(open('gpurun_out/${TAG}_${name}.json'))
print('$name', 'value %.4g'%d['value'], d['unit'], 'ms %.4f'%d['ms_per_step'], 'e2e %.4g'%d['e2e']['value'], 'roofline', d.get('roofline',{}).get('kernel'), d.get('roofline',{}).get('frac'))
" || tail -3 gpurun_out/${TAG}_${name}.err
}
run cfg2 --config 2
run cfg2_explicit --config 2 --argmax 1 --no-cpu-baseline
run cfg1 --config 1 --no-cpu-baseline
run cfg3 --config 3
run cfg4 --config 4 --steps 10 --warmup 3 --no-cpu-baseline
run cfg5 --config 5 --steps 5 --warmup 3
run reference --impl reference --steps 20 --warmup 5
