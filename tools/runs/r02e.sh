mkdir -p gpurun_out/r02e
python tools/estep_time.py scale 5 > gpurun_out/r02e/time.txt 2>&1
for v in mr152; do LSGCPD_LIB=build/diag/lib_$v.so python tools/estep_time.py scale 5 >> gpurun_out/r02e/time.txt 2>&1; done
cat gpurun_out/r02e/time.txt
