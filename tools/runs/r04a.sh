#!/bin/bash
# pairloop microbenchmark: tile-centred (mode 3) vs expanded residual (mode 4)
mkdir -p gpurun_out/r04a
cd tools/microbench && ./pairloop > ../../gpurun_out/r04a/pairloop.txt 2>&1
echo rc=$?
