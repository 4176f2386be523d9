#!/bin/bash
# pipelined last-CTA reductions + fixed-mode merge fast path: small registrations vs the previous build, tests
O=gpurun_out/r04v; mkdir -p $O; : > $O/reg.txt
for lib in build/diag/lib_base.so "" build/diag/lib_base.so ""; do
  echo "lib=$lib" >> $O/reg.txt
  LSGCPD_LIB=$lib CFGS=tiny,object,rgbd timeout 300 python tools/reg_speed.py >> $O/reg.txt 2>&1
done
cat $O/reg.txt
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.txt
