#!/bin/bash
# expanded residual: speed per mode (tile_stats on scale), E-step time, gate sweeps, E-step parity tests
O=gpurun_out/r04b; mkdir -p $O
python tools/estep_time.py scale 5 > $O/time.txt 2>&1; cat $O/time.txt
LSGCPD_EXPAND_GATE=0 python tools/estep_time.py scale 5 > $O/time_noexp.txt 2>&1; cat $O/time_noexp.txt
timeout 900 python tools/tile_stats.py scale > $O/tile_stats.txt 2>&1; tail -14 $O/tile_stats.txt
timeout 1500 python tests/tools/gate_sweep.py tiny object rgbd scale > $O/gate_sweep.txt 2>&1; cat $O/gate_sweep.txt | cut -c1-250
timeout 1500 python -m pytest tests/test_gpu_estep.py -q -x > $O/pytest.txt 2>&1; echo "pytest rc=$?"; tail -4 $O/pytest.txt
