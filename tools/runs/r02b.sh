mkdir -p gpurun_out/r02b
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader > gpurun_out/r02b/gpu.txt
timeout 900 python tools/tile_stats.py scale rgbd lidar object > gpurun_out/r02b/tile_stats.txt 2>&1; echo "tile_stats rc=$?"
timeout 1500 python -m pytest tests/test_gpu_estep.py -x -q > gpurun_out/r02b/pytest_estep.txt 2>&1; echo "pytest estep rc=$?"
timeout 600 python bench.py --steps 2 --warmup 1 --skip-cpu --skip-e2e > gpurun_out/r02b/bench.json 2> gpurun_out/r02b/bench.err; echo "bench rc=$?"
tail -3 gpurun_out/r02b/pytest_estep.txt
