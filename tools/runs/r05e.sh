#!/bin/bash
# Morton-ordered source + far-point rule: registration speed per config (sort/far on/off), then the GPU suite
O=gpurun_out/r05e; mkdir -p $O; : > $O/reg.txt
for cfg in "0 0" "1 0" "1 1" "0 1"; do
  set -- $cfg
  echo "sort_source=$1 far_rule=$2" >> $O/reg.txt
  LSGCPD_SORT_SOURCE=$1 LSGCPD_FAR_RULE=$2 CFGS=object,rgbd,lidar timeout 600 python tools/reg_speed.py >> $O/reg.txt 2>&1
done
cat $O/reg.txt | grep -v clocks
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.txt
