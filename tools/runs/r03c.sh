O=gpurun_out/r03c; mkdir -p $O
python tools/estep_time.py scale 5 > $O/time.txt 2>&1
LSGCPD_LIB=build/diag/lib_mspin.so timeout 120 python tools/estep_time.py scale 5 >> $O/time.txt 2>&1
cat $O/time.txt
