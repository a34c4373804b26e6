O=gpurun_out/r4m; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "l2_prefetch" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
