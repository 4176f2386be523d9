#!/bin/bash
# helper-warp wait variants (diagnostic builds) x residual mode (expanded product gates / centred only)
O=gpurun_out/r04d; mkdir -p $O; : > $O/time.txt
for lib in "" build/diag/lib_ns128.so build/diag/lib_ns512.so build/diag/lib_mw1.so build/diag/lib_mw1ns256.so; do
  for xg in 4 0; do
    LSGCPD_LIB=$lib LSGCPD_EXPAND_GATE=$xg timeout 300 python tools/estep_time.py scale 5 2>&1 | sed "s/^/xg=$xg /" >> $O/time.txt
  done
done
cat $O/time.txt
