#!/bin/bash
# final refresh of round 2 (after the far-point rule and the Morton-ordered sources)
TAG=r05x bash tools/refresh_profiles.sh
O=gpurun_out/r05x
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_ref.err; echo "ref rc=$?"
