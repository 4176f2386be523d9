O=gpurun_out/r03e; mkdir -p $O
python tools/estep_time.py scale 5 > $O/time.txt 2>&1
LSGCPD_LIB=build/diag/lib_punroll.so timeout 120 python tools/estep_time.py scale 5 >> $O/time.txt 2>&1
cat $O/time.txt
