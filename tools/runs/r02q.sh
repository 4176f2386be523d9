O=gpurun_out/r02q; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_register.py -q -k concurrent > $O/pytest_conc.txt 2>&1; echo "conc rc=$?"; tail -2 $O/pytest_conc.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.txt
