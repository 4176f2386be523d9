#!/bin/bash
O=gpurun_out/r04r; mkdir -p $O
LSGCPD_LIB=build/diag/lib_rb4.so timeout 150 python tools/estep_time.py scale 5 > $O/time_rb4.txt 2>&1; echo "rc=$?"; cat $O/time_rb4.txt
timeout 150 python tools/estep_time.py scale 5 > $O/time_base.txt 2>&1; cat $O/time_base.txt
