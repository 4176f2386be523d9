#!/bin/bash
O=gpurun_out/r04z; mkdir -p $O; : > $O/time.txt
for lib in "" build/diag/lib_u12.so build/diag/lib_w16u.so; do
  LSGCPD_LIB=$lib timeout 150 python tools/estep_time.py scale 5 >> $O/time.txt 2>&1
done
cat $O/time.txt
