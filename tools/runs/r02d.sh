mkdir -p gpurun_out/r02d
python tools/estep_time.py scale 5 > gpurun_out/r02d/time.txt 2>&1
for v in lag0 lag2 lag3; do LSGCPD_LIB=build/diag/lib_$v.so python tools/estep_time.py scale 5 >> gpurun_out/r02d/time.txt 2>&1; done
python tools/estep_time.py scale 5 >> gpurun_out/r02d/time.txt 2>&1
cat gpurun_out/r02d/time.txt
timeout 1500 python -m pytest tests/test_gpu_estep.py -x -q > gpurun_out/r02d/pytest_estep.txt 2>&1; echo "pytest estep rc=$?"
tail -3 gpurun_out/r02d/pytest_estep.txt
