#!/bin/bash
# Quick gpurun call: GPU parity tests + one bench line (no CPU baseline).  usage: tools/gpu_quick.sh TAG [bench args]
TAG=${1:-q}; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
tail -3 gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline "$@" > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python -c "
import json,sys
d=json.load(open('gpurun_out/${TAG}_bench.json'))
print('value',d['value'],'ms',d['ms_per_step'],'e2e',d['e2e']['value'])
print({k:round(v,4) for k,v in d['kernels_ms_per_step'].items()})
" || tail -20 gpurun_out/${TAG}_bench.err
