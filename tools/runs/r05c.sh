#!/bin/bash
O=gpurun_out/r05c; mkdir -p $O; : > $O/time.txt
for r in 1 2; do
  timeout 150 python tools/estep_time.py scale 5 2>&1 | grep "0.02" | sed 's/^/halves=2 /' >> $O/time.txt
  LSGCPD_HALVES=1 timeout 150 python tools/estep_time.py scale 5 2>&1 | grep "0.02" | sed 's/^/halves=1 /' >> $O/time.txt
done
cat $O/time.txt
