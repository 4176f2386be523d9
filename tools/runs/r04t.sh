#!/bin/bash
# merge partial loops unrolled by 16: tiny/object registration speed, vs the previous build
O=gpurun_out/r04t; mkdir -p $O
for lib in build/diag/lib_base.so "" build/diag/lib_base.so ""; do
  echo "lib=$lib" >> $O/reg.txt
  LSGCPD_LIB=$lib CFGS=tiny,object timeout 300 python tools/reg_speed.py >> $O/reg.txt 2>&1
done
cat $O/reg.txt
