#!/bin/bash
# One gpurun call that regenerates every measurement file under profiles/ for TAG (not the ncu full capture).
set -u
TAG=${TAG:-r01i}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/${TAG}_gpu.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
SHORT="python bench.py --steps 1 --warmup 1 --skip-cpu --skip-e2e --iters 3"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    $SHORT > gpurun_out/ncu_launch_${TAG}.log 2>&1; echo "launch list rc=$?"
for c in tiny object; do
  timeout 300 python bench.py --config $c --replicas --steps 20 --warmup 3 > gpurun_out/bench_${TAG}_${c}_replicas.json 2>/dev/null
done
python tools/reg_speed.py > gpurun_out/${TAG}_reg_speed.txt 2>&1
python tools/newton_cost.py >> gpurun_out/${TAG}_reg_speed.txt 2>&1
python tools/batch_speed.py > gpurun_out/${TAG}_batch_speed.txt 2>&1
python tools/cf_speed.py > gpurun_out/${TAG}_cf_speed.txt 2>&1
python tools/ext_speed.py > gpurun_out/${TAG}_ext_speed.txt 2>&1
python tools/prep_speed.py > gpurun_out/${TAG}_prep_speed.txt 2>&1
python tools/golden_errors.py > gpurun_out/${TAG}_golden_errors.txt 2>&1
python tools/small_path_sweep.py > gpurun_out/${TAG}_small_path_sweep.txt 2>&1
echo done
