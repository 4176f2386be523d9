O=gpurun_out/r02r; mkdir -p $O
python tools/estep_time.py scale 5 > $O/time.txt 2>&1
LSGCPD_LIB=build/diag/lib_w16.so python tools/estep_time.py scale 5 >> $O/time.txt 2>&1
cat $O/time.txt
LSGCPD_LIB=build/diag/lib_w16.so timeout 900 python -m pytest tests/test_gpu_estep.py -q -x -k "tensor_core_and_cuda_core or sampled_parity_at_full_scale or ragged" > $O/pytest_w16.txt 2>&1; echo "w16 pytest rc=$?"
tail -2 $O/pytest_w16.txt
