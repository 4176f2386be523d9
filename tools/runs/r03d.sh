O=gpurun_out/r03d; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_batch.py -q > $O/pytest.txt 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.txt
tools/with_clocks.sh $O/batch_speed.txt python tools/batch_speed.py; tail -4 $O/batch_speed.txt
