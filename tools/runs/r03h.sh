TAG=r03h bash tools/refresh_profiles.sh
O=gpurun_out/r03h
SHORT="python bench.py --steps 1 --warmup 1 --skip-cpu --skip-e2e --iters 3"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:estep_tc_kernel -s 1 -c 1 -o $O/estep_full $SHORT > $O/ncu_full.log 2>&1; echo "ncu rc=$?"
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gpu.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
