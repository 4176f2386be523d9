O=gpurun_out/r02s; mkdir -p $O
LSGCPD_LIB=build/diag/lib_w16.so timeout 120 python tools/estep_time.py scale 5 > $O/time.txt 2>&1; echo "w16 rc=$?"
cat $O/time.txt
LSGCPD_LIB=build/diag/lib_w16.so timeout 300 python -m pytest tests/test_gpu_estep.py -q -x -k "tensor_core_and_cuda_core or ragged" > $O/pytest_w16.txt 2>&1; echo "w16 pytest rc=$?"
tail -2 $O/pytest_w16.txt
