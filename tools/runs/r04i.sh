#!/bin/bash
O=gpurun_out/r04i; mkdir -p $O
timeout 600 python tools/prep_batch_time.py 550 3500 5 > $O/prep_batch.txt 2>&1; cat $O/prep_batch.txt
timeout 600 python tools/prep_batch_time.py 64 20000 3 >> $O/prep_batch.txt 2>&1; tail -3 $O/prep_batch.txt
timeout 1200 python -m pytest tests/test_gpu_batch.py tests/test_gpu_prepare.py -q > $O/pytest.txt 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.txt
