#!/bin/bash
# after the batched prepare: full GPU suite, smoke, batch bench line, batch speed
O=gpurun_out/r04m; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.txt
timeout 900 python bench.py --config batch > $O/bench_batch.json 2> $O/bench_batch.err; echo "batch bench rc=$?"
bash tools/with_clocks.sh $O/batch_speed.txt python tools/batch_speed.py; cat $O/batch_speed.txt
