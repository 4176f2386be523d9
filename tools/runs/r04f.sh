#!/bin/bash
# batched E step: register split of the batch tensor-core kernel (diagnostic builds) vs the product
O=gpurun_out/r04f; mkdir -p $O; : > $O/batch.txt
for lib in "" build/diag/lib_bt152.so build/diag/lib_bt160.so ""; do
  echo "lib=$lib" >> $O/batch.txt
  LSGCPD_LIB=$lib timeout 600 python tools/batch_speed.py 2>&1 | grep "batch B" >> $O/batch.txt
done
cat $O/batch.txt
