O=gpurun_out/r02m; mkdir -p $O
SHORT="python bench.py --steps 1 --warmup 1 --skip-cpu --skip-e2e --iters 3"
timeout 600 $SHORT > $O/short.log 2>&1; echo "short rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:estep_tc_kernel -s 1 -c 1 \
    -o $O/estep_full $SHORT > $O/ncu_full.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"morton|slot_inverse|pack_|RadixSort" -c 8 -o $O/pack_scale \
    python tools/secondary_once.py scale 1 > $O/ncu_pack.log 2>&1; echo "pack rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_scale_prep.csv \
    python tools/secondary_once.py scale 2 > $O/ncu_l.log 2>&1; echo "launch rc=$?"
