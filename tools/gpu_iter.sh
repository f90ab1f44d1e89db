#!/bin/bash
# Iteration gpurun call: selected GPU tests (pytest -k EXPR, or all), cfg 2 and cfg 4 bench lines.
# usage: tools/gpu_iter.sh TAG [pytest -k expression]
TAG=${1:-it}; K=${2:-}
mkdir -p gpurun_out
if [ -n "$K" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/${TAG}_pytest_gpu.log 2>&1
else
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1
fi
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
tail -4 gpurun_out/${TAG}_pytest_gpu.log
for args in "--config 2" "--config 4 --steps 5 --warmup 3"; do
  name=$(echo $args | tr -d ' -')
  timeout 600 python bench.py --no-cpu-baseline $args > gpurun_out/${TAG}_${name}.json 2> gpurun_out/${TAG}_${name}.err
  python -c "
import json
d=json.load(open('gpurun_out/${TAG}_${name}.json'))
print('$name', 'value %.4g'%d['value'], 'ms %.4f'%d['ms_per_step'], 'e2e %.4g'%d['e2e']['value'], {k:round(v,4) for k,v in d['kernels_ms_per_step'].items()})
" || tail -5 gpurun_out/${TAG}_${name}.err
done
