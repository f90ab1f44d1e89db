#!/bin/bash
# A/B of an environment switch: tools-less inline.  usage: abenv.sh TAG "bench args" "ENVA" "ENVB"
TAG=$1; ARGS=$2
for v in "$3" "$4"; do
  for rep in 1 2; do
    env $v timeout 600 python bench.py --no-cpu-baseline $ARGS > gpurun_out/${TAG}_$rep.json 2> gpurun_out/${TAG}_$rep.err
    python -c "
import json
d=json.load(open('gpurun_out/${TAG}_$rep.json'))
print('$v $rep', 'ms %.4f'%d['ms_per_step'], {k:round(v,4) for k,v in d['kernels_ms_per_step'].items()})
" || tail -5 gpurun_out/${TAG}_$rep.err
  done
done
