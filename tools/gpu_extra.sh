#!/bin/bash
# Supplementary bench lines: config 3 (brute force) and config 5 (inference).  usage: tools/gpu_extra.sh TAG
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 python bench.py --config 3 --steps 5 --warmup 3 --cpu-seconds 10 > gpurun_out/${TAG}_cfg3.json 2> gpurun_out/${TAG}_cfg3.err; tail -c 1500 gpurun_out/${TAG}_cfg3.json; tail -3 gpurun_out/${TAG}_cfg3.err
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 > gpurun_out/${TAG}_cfg5.json 2> gpurun_out/${TAG}_cfg5.err; tail -c 1500 gpurun_out/${TAG}_cfg5.json; tail -3 gpurun_out/${TAG}_cfg5.err
