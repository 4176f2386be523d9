O=gpurun_out/r03g; mkdir -p $O
python tools/estep_time.py scale 5 > $O/time.txt 2>&1
LSGCPD_LIB=build/diag/lib_ssm.so timeout 120 python tools/estep_time.py scale 5 >> $O/time.txt 2>&1
cat $O/time.txt
LSGCPD_LIB=build/diag/lib_ssm.so timeout 300 python -m pytest tests/test_gpu_estep.py -q -x -k "tensor_core_and_cuda_core or sampled_parity_at_full_scale or ragged" > $O/pytest.txt 2>&1; echo "rc=$?"; tail -1 $O/pytest.txt
