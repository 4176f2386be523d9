#!/bin/bash
# warm-cache per-kernel durations of short tiny/object registrations (small-problem tail analysis)
O=gpurun_out/r04s; mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file $O/launches.csv python tools/small_reg_once.py > $O/ncu.log 2>&1; echo "rc=$?"
python tools/launch_shares.py $O/launches.csv > $O/shares.txt; cat $O/shares.txt | head -30
