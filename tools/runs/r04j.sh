#!/bin/bash
# wave-batched lsgcpd_prepare_batch: byte-for-byte tests, batch parity, timings
O=gpurun_out/r04j; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_prepare.py tests/test_gpu_batch.py -q -x > $O/pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.txt
timeout 600 python tools/prep_batch_time.py 550 3500 5 > $O/prep_batch.txt 2>&1; cat $O/prep_batch.txt
timeout 600 python tools/prep_batch_time.py 64 20000 3 >> $O/prep_batch.txt 2>&1; tail -3 $O/prep_batch.txt
timeout 600 python tools/prep_batch_time.py 4 200000 3 >> $O/prep_batch.txt 2>&1; tail -3 $O/prep_batch.txt
bash tools/with_clocks.sh $O/batch_speed.txt python tools/batch_speed.py; cat $O/batch_speed.txt
