#!/bin/bash
# ncu --set full of estep_tc_kernel: expanded residual (product gates) vs centred only
O=gpurun_out/r04c; mkdir -p $O
SHORT="python bench.py --steps 1 --warmup 1 --skip-cpu --skip-e2e --iters 3"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:estep_tc_kernel -s 1 -c 1 -o $O/exp $SHORT > $O/ncu_exp.log 2>&1; echo "ncu rc=$?"
LSGCPD_EXPAND_GATE=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:estep_tc_kernel -s 1 -c 1 -o $O/cen $SHORT > $O/ncu_cen.log 2>&1; echo "ncu rc=$?"
