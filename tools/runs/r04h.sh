#!/bin/bash
O=gpurun_out/r04h; mkdir -p $O
timeout 600 python tools/prep_batch_time.py 550 3500 5 > $O/prep_batch.txt 2>&1; cat $O/prep_batch.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/prep_launches.csv python tools/prep_batch_time.py 20 3500 1 > $O/ncu.log 2>&1; echo "ncu rc=$?"
python tools/launch_shares.py $O/prep_launches.csv > $O/prep_shares.txt 2>&1; cat $O/prep_shares.txt | head -40
