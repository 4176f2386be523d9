#!/bin/bash
# FFMA / FFMA2 / MUFU.EX2 pipe rates on the box with the SM clock sampled during the runs (nvidia-smi every
# 100 ms) and the in-kernel clock64 estimate; writes gpurun_out/$TAG/pipes.txt and pipes_clocks.csv.
set -u
TAG=${TAG:-r02}
O=gpurun_out/$TAG; mkdir -p $O
cd "$(dirname "$0")"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes pipes.cu || exit 1
cd - > /dev/null
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv,noheader,nounits -lms 100 > $O/pipes_clocks.csv &
SMI=$!
for i in $(seq 1 15); do tools/microbench/pipes; done > $O/pipes.txt
kill $SMI
