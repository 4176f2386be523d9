TAG=r02w bash tools/refresh_profiles.sh
O=gpurun_out/r02w
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.txt
