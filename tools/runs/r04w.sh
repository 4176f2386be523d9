#!/bin/bash
# ncu --set full of em_tail_kernel on tiny and object (warm caches)
O=gpurun_out/r04w; mkdir -p $O
for c in tiny object; do
  timeout 600 ncu --set full --clock-control none --cache-control none --import-source on -k regex:em_tail -c 1 -s 2 -o $O/emtail_$c \
    python tools/secondary_once.py $c 4 > $O/ncu_$c.log 2>&1; echo "$c rc=$?"
done
