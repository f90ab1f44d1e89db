#!/bin/bash
# Round-2 gpurun call: host info, GPU parity tests (no -x: every failure listed), smoke, bench.
# usage: tools/gpu_r2.sh TAG [pytest -k expr]
TAG=${1:-r2}; K=${2:-}
mkdir -p gpurun_out
{ nproc; python -c "import os; print('affinity', len(os.sched_getaffinity(0)))"; grep -m1 "model name" /proc/cpuinfo;
  nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; } > gpurun_out/${TAG}_host.txt 2>&1
export HRP_PARITY_LOG=$PWD/gpurun_out/${TAG}_parity.jsonl
rm -f $HRP_PARITY_LOG
if [ -n "$K" ]; then KA=(-k "$K"); else KA=(); fi
timeout 3000 python -m pytest tests -m gpu -q -rfE --durations=25 "${KA[@]}" > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest_gpu.log
tail -40 gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
tail -2 gpurun_out/${TAG}_smoke.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python -c "
import json
d=json.load(open('gpurun_out/${TAG}_bench.json'))
print('value',d['value'],'ms',d['ms_per_step'],'e2e',d['e2e']['value'], 'cpu', d.get('cpu_baseline'))
print({k:round(v,4) for k,v in d['kernels_ms_per_step'].items()})
" || tail -20 gpurun_out/${TAG}_bench.err
