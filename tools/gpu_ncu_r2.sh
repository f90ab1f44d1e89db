#!/bin/bash
# ncu evidence for round 2: cfg2 bench launch list (time + DRAM bytes per launch), full captures
# of the cfg4 selection / TD kernels and of the cfg2 hidden-layer GEMM.
TAG=${1:-r2o}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -c 600 --csv --log-file gpurun_out/${TAG}_launches_cfg2.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:sel_kernel" -s 2 -c 1 \
  -o gpurun_out/${TAG}_sel_cfg4 python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline \
  > gpurun_out/${TAG}_ncu_sel.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:td_kernel" -s 2 -c 1 \
  -o gpurun_out/${TAG}_td_cfg4 python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline \
  > gpurun_out/${TAG}_ncu_td.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:tc_gemm_kernel" -s 40 -c 1 \
  -o gpurun_out/${TAG}_gemm_cfg2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
  > gpurun_out/${TAG}_ncu_gemm.log 2>&1
ls -la gpurun_out | grep $TAG
