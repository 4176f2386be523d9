#!/bin/bash
# 16 consumer warps (4 warpgroups, 2 MMA warps, 112 registers) vs the product
O=gpurun_out/r04e; mkdir -p $O; : > $O/time.txt
for lib in "" build/diag/lib_w16.so; do
  LSGCPD_LIB=$lib timeout 300 python tools/estep_time.py scale 5 >> $O/time.txt 2>&1
done
cat $O/time.txt
