O=gpurun_out/r4p; mkdir -p $O
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_filter.py tests/test_gpu_upload.py tests/test_gpu_dist.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for r in 1 2; do timeout 300 python tools/c3_phases.py >> $O/phases.txt 2>&1; done
