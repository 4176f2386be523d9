O=gpurun_out/r02z3; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_fullscale.py -q -k "teacher_forced" --durations=3 > $O/pytest.txt 2>&1; echo "rc=$?"; tail -8 $O/pytest.txt
