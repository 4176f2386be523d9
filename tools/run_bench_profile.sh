#!/bin/bash
# One gpurun call: bench (default), then a short plain run + ncu launch list + ncu full capture of the E step.
set -u
mkdir -p gpurun_out
TAG=${TAG:-r01}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_${TAG}.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_${TAG}.json
SHORT="python bench.py --steps 1 --warmup 1 --skip-cpu --skip-e2e --iters 3"
if [ "${NCU:-1}" = "1" ]; then
  timeout 600 $SHORT > gpurun_out/short_${TAG}.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_${TAG}.csv $SHORT > gpurun_out/ncu_launch_${TAG}.log 2>&1
  echo "launch list rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-estep_tc_kernel} -s 1 -c ${NCU_COUNT:-2} \
      -o gpurun_out/prof_estep_${TAG} $SHORT > gpurun_out/ncu_full_${TAG}.log 2>&1
  echo "ncu full rc=$?"
fi
