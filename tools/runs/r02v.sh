O=gpurun_out/r02v; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fullscale.py -q -k "without_graph or one_rank" > $O/pytest.txt 2>&1; echo "rc=$?"; tail -3 $O/pytest.txt
