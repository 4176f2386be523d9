O=gpurun_out/r03b; mkdir -p $O
python tools/estep_time.py scale 5 > $O/time.txt 2>&1; cat $O/time.txt
timeout 900 python -m pytest tests/test_gpu_estep.py tests/test_gpu_register.py -q -x > $O/pytest.txt 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.txt
