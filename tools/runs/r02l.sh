O=gpurun_out/r02l; mkdir -p $O
python tools/estep_time.py scale 5 > $O/time.txt 2>&1
for v in early nt8; do LSGCPD_LIB=build/diag/lib_$v.so python tools/estep_time.py scale 5 >> $O/time.txt 2>&1; done
cat $O/time.txt
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?"
tail -3 $O/pytest_gpu.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
