#!/bin/bash
# A/B of prebuilt libhrp variants (ab/libhrp_<name>.so): one bench line per variant and config.
# usage: tools/gpu_ab.sh TAG "bench args" name1 name2 ...
TAG=$1; ARGS=$2; shift; shift
mkdir -p gpurun_out
cp paper_2405_08754_b200/libhrp.so /tmp/libhrp_orig.so
for v in "$@"; do
  cp ab/libhrp_$v.so paper_2405_08754_b200/libhrp.so
  for rep in 1 2; do
    timeout 600 python bench.py --no-cpu-baseline $ARGS > gpurun_out/${TAG}_${v}_$rep.json 2> gpurun_out/${TAG}_${v}_$rep.err
    python -c "
import json
d=json.load(open('gpurun_out/${TAG}_${v}_$rep.json'))
print('$v $rep', 'ms %.4f'%d['ms_per_step'], {k:round(v,4) for k,v in d['kernels_ms_per_step'].items()})
" || tail -5 gpurun_out/${TAG}_${v}_$rep.err
  done
done
cp /tmp/libhrp_orig.so paper_2405_08754_b200/libhrp.so
