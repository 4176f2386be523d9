#!/bin/bash
# One gpurun call: ncu launch lists of prepare + short registrations (object / lidar / scale) and one
# `ncu --set full` capture per secondary kernel family (kNN + surface fit, em_tail / moments, Newton).
set -u
mkdir -p gpurun_out
TAG=${TAG:-r02a}
O=gpurun_out/sec_${TAG}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > $O/gpu.txt 2>&1
for c in object lidar scale; do
  it=5; [ $c = scale ] && it=2
  timeout 300 python tools/secondary_once.py $c $it > $O/plain_$c.log 2>&1 || { echo "plain $c failed"; cat $O/plain_$c.log; continue; }
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$c.csv \
      python tools/secondary_once.py $c $it > $O/ncu_launch_$c.log 2>&1; echo "launch list $c rc=$?"
done
# full captures: kNN kernels on lidar and scale, em_tail on object, moments + newton on scale
timeout 900 ncu --set full --clock-control none --import-source on -k regex:knn -c 3 -o $O/knn_lidar \
    python tools/secondary_once.py lidar 1 > $O/ncu_knn_lidar.log 2>&1; echo "knn lidar rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pack_|cloud_stats|model_stats|header" -c 4 -o $O/pack_scale \
    python tools/secondary_once.py scale 1 > $O/ncu_pack_scale.log 2>&1; echo "pack scale rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:knn -c 3 -o $O/knn_scale \
    python tools/secondary_once.py scale 1 > $O/ncu_knn_scale.log 2>&1; echo "knn scale rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:em_tail -c 1 -s 1 -o $O/emtail_object \
    python tools/secondary_once.py object 3 > $O/ncu_emtail_object.log 2>&1; echo "em_tail rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"moments_kernel|newton_kernel|estep_merge" -c 3 -s 3 -o $O/mstep_scale \
    python tools/secondary_once.py scale 2 > $O/ncu_mstep_scale.log 2>&1; echo "mstep scale rc=$?"
ls -la $O
