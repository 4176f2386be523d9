#!/bin/bash
# ncu --set full of the final estep_tc_kernel (far-point rule build), one half-sweep of scale
O=gpurun_out/r05j; mkdir -p $O
SHORT="python bench.py --steps 1 --warmup 1 --skip-cpu --skip-e2e --iters 3"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:estep_tc_kernel -s 1 -c 1 -o $O/estep_full $SHORT > $O/ncu_full.log 2>&1; echo "ncu rc=$?"
