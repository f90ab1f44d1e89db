#!/bin/bash
# Final evidence of a change: GPU tests, bench lines (cfg 1, 2, 2 pruned, 4, 5), the cfg 2 and
# cfg 4 ncu launch lists (time + DRAM bytes per launch).  usage: tools/gpu_round_end.sh TAG
TAG=${1:-e}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
tail -3 gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench_cfg2.json 2> gpurun_out/${TAG}_bench_cfg2.err
for args in "--config 2 --argmax 2" "--config 1" "--config 4 --steps 5 --warmup 3" "--config 5 --steps 3 --warmup 3"; do
  name=$(echo $args | tr -d ' -')
  timeout 900 python bench.py --no-cpu-baseline $args > gpurun_out/${TAG}_${name}.json 2> gpurun_out/${TAG}_${name}.err
done
for f in gpurun_out/${TAG}_*.json; do
  python -c "
import json,sys
d=json.load(open('$f'))
print('$f', 'value %.4g'%d['value'], 'ms %.4f'%d['ms_per_step'], 'e2e %.4g'%d['e2e']['value'], d.get('kernels_ms_per_step',''))
" || tail -3 ${f%.json}.err
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -c 600 --csv \
  --log-file gpurun_out/${TAG}_launches_cfg2.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline \
  > gpurun_out/${TAG}_ncu_cfg2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -c 400 --csv \
  --log-file gpurun_out/${TAG}_launches_cfg4.csv python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline \
  > gpurun_out/${TAG}_ncu_cfg4.log 2>&1
ls gpurun_out | grep ${TAG}
