#!/bin/bash
# One ncu --set full capture of kernels matching $2 in a short bench run.  usage: tools/gpu_ncu1.sh TAG REGEX [bench args]
TAG=$1; K=$2; shift; shift
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$K" -s 6 -c 1 \
  -o gpurun_out/${TAG}_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/${TAG}_ncu.log 2>&1
tail -3 gpurun_out/${TAG}_ncu.log
