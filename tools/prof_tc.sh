#!/bin/bash
# ncu full capture of the tensor-core E step on the scale config (plain run first).
TAG=${TAG:-tc}
export CFG=${CFG:-scale}
python tools/estep_once.py > gpurun_out/once_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-estep_tc_kernel} -s 1 -c 1 -o gpurun_out/prof_${TAG} python tools/estep_once.py > gpurun_out/ncu_${TAG}.log 2>&1
tail -1 gpurun_out/ncu_${TAG}.log
