#!/bin/bash
O=gpurun_out/r05b; mkdir -p $O; : > $O/time.txt
for r in 1 2; do for lib in "" build/diag/lib_adb.so; do
  LSGCPD_LIB=$lib timeout 150 python tools/estep_time.py scale 5 2>&1 | grep "0.02" >> $O/time.txt
done; done
cat $O/time.txt
LSGCPD_LIB=build/diag/lib_adb.so timeout 900 python -m pytest tests/test_gpu_estep.py -q -x -k "sigma_sweep or ragged" > $O/pytest.txt 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.txt
