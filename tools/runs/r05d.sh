#!/bin/bash
# far-point rule: speed (registrations, batch, E step per config) and precision (gate sweep), rule on vs off
O=gpurun_out/r05d; mkdir -p $O
for fr in 0 1; do
  LSGCPD_FAR_RULE=$fr CFGS=tiny,object,rgbd,lidar timeout 600 python tools/reg_speed.py > $O/reg_far$fr.txt 2>&1
  LSGCPD_FAR_RULE=$fr timeout 600 python tools/batch_speed.py > $O/batch_far$fr.txt 2>&1
done
cat $O/reg_far0.txt $O/reg_far1.txt $O/batch_far0.txt $O/batch_far1.txt | grep -v clocks
timeout 2400 python tests/tools/gate_sweep.py tiny object rgbd lidar > $O/gate_sweep.txt 2>&1; cut -c1-220 $O/gate_sweep.txt
