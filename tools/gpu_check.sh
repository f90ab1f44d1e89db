#!/bin/bash
# One gpurun call: GPU parity tests, the bench line, the ncu launch list (time + DRAM bytes per
# launch) and full captures.  usage: tools/gpu_check.sh TAG [full-capture kernel regexes...]
set -x
TAG=${1:-v}; shift
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -c 600 --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline \
  > gpurun_out/${TAG}_ncu_bench.log 2>&1
for K in "$@"; do
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$K" -s 6 -c 1 \
    -o gpurun_out/${TAG}_full_${K//[^a-zA-Z0-9]/_} python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
    > gpurun_out/${TAG}_ncu_full_${K//[^a-zA-Z0-9]/_}.log 2>&1
done
ls -la gpurun_out
