O=gpurun_out/r02h; mkdir -p $O
python tools/estep_time.py scale 5 > $O/time.txt 2>&1
LSGCPD_LIB=build/diag/lib_paired.so python tools/estep_time.py scale 5 >> $O/time.txt 2>&1
cat $O/time.txt
LSGCPD_LIB=build/diag/lib_paired.so timeout 900 python -m pytest tests/test_gpu_estep.py -q -x -k "tensor_core_and_cuda_core or sampled_parity_at_full_scale or ragged" > $O/pytest_paired.txt 2>&1; echo "paired pytest rc=$?"
tail -2 $O/pytest_paired.txt
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?"
tail -4 $O/pytest_gpu.txt
