mkdir -p gpurun_out/r02c
timeout 1200 python tests/tools/gate_sweep.py > gpurun_out/r02c/gate_sweep.txt 2>&1; echo "sweep rc=$?"
SHORT="python bench.py --steps 1 --warmup 1 --skip-cpu --skip-e2e --iters 3"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:estep_tc_kernel -s 1 -c 1 \
    -o gpurun_out/r02c/estep_full $SHORT > gpurun_out/r02c/ncu_full.log 2>&1; echo "ncu rc=$?"
