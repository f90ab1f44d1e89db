#!/bin/bash
# peaks + compute-sanitizer (memcheck, racecheck, synccheck) on config 1 + cfg4/cfg3 bench lines
mkdir -p gpurun_out
timeout 300 python tools/measure_peaks.py > gpurun_out/r2f_peaks.log 2>&1
for T in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $T --print-limit 50 python tools/sanitize_cfg1.py > gpurun_out/r2f_sanitize_$T.log 2>&1
  echo "rc=$?" >> gpurun_out/r2f_sanitize_$T.log
done
timeout 600 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2f_bench_cfg4.json 2> gpurun_out/r2f_bench_cfg4.err
timeout 600 python bench.py --config 3 --no-cpu-baseline > gpurun_out/r2f_bench_cfg3.json 2> gpurun_out/r2f_bench_cfg3.err
tail -3 gpurun_out/r2f_sanitize_*.log
