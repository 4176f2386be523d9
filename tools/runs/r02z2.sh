O=gpurun_out/r02z2; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_estep.py -q -k "sampled_parity_at_full_scale and default-auto" --durations=3 > $O/pytest.txt 2>&1; echo "rc=$?"; tail -6 $O/pytest.txt
