#!/bin/bash
# One gpurun call that regenerates the measurement files of a round under gpurun_out/$TAG (then copied to
# profiles/$TAG by hand): bench (scale, default), the ncu launch list of a short bench, the replicas benches,
# and every speed tool with the SM clock sampled under load (tools/with_clocks.sh).
set -u
TAG=${TAG:-r02}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > $O/gpu.txt 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
SHORT="python bench.py --steps 1 --warmup 1 --skip-cpu --skip-e2e --iters 3"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    $SHORT > $O/ncu_launch.log 2>&1; echo "launch list rc=$?"
for c in tiny object; do
  timeout 300 python bench.py --config $c --replicas --steps 20 --warmup 3 > $O/bench_${c}_replicas.json 2>/dev/null
done
timeout 900 python bench.py --config batch > $O/bench_batch.json 2> $O/bench_batch.err; echo "batch bench rc=$?"
W=tools/with_clocks.sh
$W $O/reg_speed.txt python tools/reg_speed.py
$W $O/newton_cost.txt python tools/newton_cost.py
$W $O/batch_speed.txt python tools/batch_speed.py
$W $O/cf_speed.txt python tools/cf_speed.py
$W $O/ext_speed.txt python tools/ext_speed.py
$W $O/prep_speed.txt python tools/prep_speed.py
$W $O/shard_speed.txt python tools/shard_speed.py
$W $O/tile_stats.txt python tools/tile_stats.py
$W $O/golden_errors.txt python tools/golden_errors.py
$W $O/small_path_sweep.txt python tools/small_path_sweep.py
echo done
