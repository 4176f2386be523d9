O=gpurun_out/r02z4; mkdir -p $O
timeout 2400 python -m pytest tests/test_gpu_affine.py tests/test_gpu_model_ext.py tests/test_gpu_fullscale.py -q > $O/pytest.txt 2>&1; echo "rc=$?"; tail -4 $O/pytest.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.txt
