O=gpurun_out/r02i; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?"
tail -4 $O/pytest_gpu.txt
TAG=r02i bash tools/refresh_profiles.sh
