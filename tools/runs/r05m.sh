#!/bin/bash
# far-point rule threshold: d >= 2 R (product), 1.5 R, 1.2 R — lidar/rgbd speed and precision
O=gpurun_out/r05m; mkdir -p $O; : > $O/reg.txt; : > $O/sweep.txt
for lib in "" build/diag/lib_k15.so build/diag/lib_k12.so; do
  echo "lib=$lib" >> $O/reg.txt
  LSGCPD_LIB=$lib CFGS=rgbd,lidar timeout 600 python tools/reg_speed.py 2>&1 | grep -v clocks >> $O/reg.txt
  echo "lib=$lib" >> $O/sweep.txt
  LSGCPD_LIB=$lib timeout 1500 python tests/tools/gate_sweep.py rgbd lidar 2>&1 | grep "G+far" >> $O/sweep.txt
done
cat $O/reg.txt; cut -c1-150 $O/sweep.txt
