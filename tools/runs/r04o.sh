#!/bin/bash
# helper-free tensor-core kernel (LSGCPD_TC_SELF=1): timing, then E-step parity
O=gpurun_out/r04o; mkdir -p $O
LSGCPD_TC_SELF=1 timeout 120 python tools/estep_time.py scale 5 > $O/time_self.txt 2>&1; echo "self rc=$?"; cat $O/time_self.txt
timeout 120 python tools/estep_time.py scale 5 > $O/time_base.txt 2>&1; cat $O/time_base.txt
LSGCPD_TC_SELF=1 timeout 900 python -m pytest tests/test_gpu_estep.py -q -x > $O/pytest_estep.txt 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_estep.txt
