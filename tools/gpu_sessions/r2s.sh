O=gpurun_out/r2s; mkdir -p $O
timeout 2000 python -m pytest tests/test_gpu_filter.py tests/test_gpu_golden.py tests/test_gpu_parity.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python tools/filter_sweep.py c4 "" > $O/sweep_c4.txt 2>&1
