O=gpurun_out/r02t; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_estep.py -q -x -k "zero_crossing or tensor_core_and_cuda" > $O/pytest.txt 2>&1; echo "rc=$?"; tail -3 $O/pytest.txt
