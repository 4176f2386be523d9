mkdir -p gpurun_out/r02f
python tools/estep_time.py scale 5 > gpurun_out/r02f/time.txt 2>&1
for v in mr u2 mr_u2 rb3; do LSGCPD_LIB=build/diag/lib_$v.so python tools/estep_time.py scale 5 >> gpurun_out/r02f/time.txt 2>&1; done
cat gpurun_out/r02f/time.txt
