#!/bin/bash
O=gpurun_out/r04p; mkdir -p $O
LSGCPD_LIB=build/diag/lib_s16.so LSGCPD_TC_SELF=1 timeout 120 python tools/estep_time.py scale 5 > $O/time_s16.txt 2>&1; echo "rc=$?"; cat $O/time_s16.txt
