O=gpurun_out/r02y; mkdir -p $O
LSGCPD_LIB=build/diag/lib_pipe.so timeout 120 python tools/estep_time.py scale 5 > $O/time.txt 2>&1; echo "pipe rc=$?"
cat $O/time.txt
LSGCPD_LIB=build/diag/lib_pipe.so timeout 300 python -m pytest tests/test_gpu_estep.py -q -x -k "tensor_core_and_cuda_core or ragged or sampled_parity_at_full_scale" > $O/pytest.txt 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.txt
