#!/bin/bash
# A/B of programmatic dependent launch on the GEMMs + GPU tests + schedule-quality report.
# usage: tools/gpu_pdl_ab.sh TAG
TAG=${1:-p}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
tail -3 gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python tools/schedule_quality.py --out gpurun_out/${TAG}_schedule_quality.md > gpurun_out/${TAG}_sq.log 2>&1; tail -20 gpurun_out/${TAG}_sq.log
for rep in 1 2; do
  for pdl in 0 1; do
    for args in "--config 2" "--config 2 --argmax 2" "--config 4 --steps 5 --warmup 3"; do
      name=$(echo $args | tr -d ' -')_pdl${pdl}_${rep}
      if [ $pdl = 0 ]; then export HRP_NO_PDL=1; else unset HRP_NO_PDL; fi
      timeout 600 python bench.py --no-cpu-baseline $args > gpurun_out/${TAG}_${name}.json 2> gpurun_out/${TAG}_${name}.err
      python -c "
import json
d=json.load(open('gpurun_out/${TAG}_${name}.json'))
print('$name', 'ms %.4f'%d['ms_per_step'], 'e2e %.4g'%d['e2e']['value'], {k:round(v,4) for k,v in d['kernels_ms_per_step'].items() if k.startswith('gemm')})
" || tail -5 gpurun_out/${TAG}_${name}.err
    done
  done
done
