#!/bin/bash
O=gpurun_out/r05h; mkdir -p $O; : > $O/bench.txt
for r in 1 2; do for ss in 0 1; do
  LSGCPD_SORT_SOURCE=$ss timeout 600 python bench.py --steps 3 --warmup 1 --skip-cpu --skip-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('sort_source=$ss', d['value'], d['ms_per_step'])" >> $O/bench.txt
done; done
cat $O/bench.txt
