#!/bin/bash
# ncu full capture of one tensor-core E-step launch on the scale config (plain run first).
TAG=${TAG:-tc2}
export CFG=${CFG:-scale} REPS=${REPS:-2}
mkdir -p gpurun_out
python tools/estep_once.py > gpurun_out/once_${TAG}.log 2>&1 || { echo "plain run failed"; cat gpurun_out/once_${TAG}.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-estep_tc} -s 1 -c 1 \
    -o gpurun_out/prof_${TAG} python tools/estep_once.py > gpurun_out/ncu_${TAG}.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_${TAG}.log
