O=gpurun_out/r02x; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_estep.py tests/test_gpu_batch.py -q -k "literal" > $O/pytest.txt 2>&1; echo "rc=$?"; tail -3 $O/pytest.txt
