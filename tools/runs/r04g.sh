#!/bin/bash
# batch register split 152/48: parity tests, batch bench line, batch speed with clocks
O=gpurun_out/r04g; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_batch.py -q > $O/pytest_batch.txt 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_batch.txt
timeout 900 python bench.py --config batch > $O/bench_batch.json 2> $O/bench_batch.err; echo "batch bench rc=$?"; tail -c 600 $O/bench_batch.json
bash tools/with_clocks.sh $O/batch_speed.txt python tools/batch_speed.py; cat $O/batch_speed.txt
