#!/bin/bash
# midpoint tile centres with rounded y' + abs-y block for the hi/lo residual: speed and precision
O=gpurun_out/r05i; mkdir -p $O
timeout 200 python tools/estep_time.py scale 5 > $O/time.txt 2>&1; cat $O/time.txt
CFGS=tiny,object,rgbd,lidar timeout 600 python tools/reg_speed.py > $O/reg.txt 2>&1; grep -v clocks $O/reg.txt
timeout 600 python tools/batch_speed.py > $O/batch.txt 2>&1; grep "batch B" $O/batch.txt
timeout 300 python tools/tile_centre_stats.py > $O/centres.txt 2>&1; cat $O/centres.txt
timeout 1500 python -m pytest tests/test_gpu_estep.py -q -x > $O/pytest_estep.txt 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_estep.txt
timeout 2400 python tests/tools/gate_sweep.py tiny object rgbd lidar > $O/gate_sweep.txt 2>&1; cut -c1-200 $O/gate_sweep.txt
