#!/bin/bash
O=gpurun_out/r04l; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_prepare.py tests/test_gpu_batch.py -q > $O/pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.txt
for i in 1 2 3; do timeout 1200 python -m pytest tests/test_gpu_prepare.py -q -k batch >> $O/pytest_rep.txt 2>&1; done; grep -c passed $O/pytest_rep.txt; grep failed $O/pytest_rep.txt
timeout 600 python tools/prep_batch_time.py 550 3500 3 > $O/prep_batch.txt 2>&1; cat $O/prep_batch.txt
