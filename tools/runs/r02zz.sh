O=gpurun_out/r02zz; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q --durations=8 > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -14 $O/pytest_gpu.txt
