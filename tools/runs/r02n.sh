O=gpurun_out/r02n; mkdir -p $O
python tools/estep_time.py scale 5 > $O/time.txt 2>&1
for v in notc noex2 notc_noex2; do LSGCPD_LIB=build/diag/lib_$v.so python tools/estep_time.py scale 5 >> $O/time.txt 2>&1; done
cat $O/time.txt
