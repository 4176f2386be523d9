#!/bin/bash
# producer / MMA-warp wait variants (diagnostic builds) vs the product, twice each
O=gpurun_out/r05a; mkdir -p $O; : > $O/time.txt
for r in 1 2; do
for lib in "" build/diag/lib_p500.so build/diag/lib_p2k.so build/diag/lib_m32.so build/diag/lib_m32p500.so; do
  LSGCPD_LIB=$lib timeout 150 python tools/estep_time.py scale 5 2>&1 | grep "0.02" >> $O/time.txt
done
done
cat $O/time.txt
