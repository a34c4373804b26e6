O=gpurun_out/r2o; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_filter.py tests/test_gpu_golden.py tests/test_gpu_upload.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python tools/filter_sweep.py c5 "" LSAPGPU_FILTER_RB=1 > $O/sweep_c5.txt 2>&1
timeout 900 python tools/filter_sweep.py c4 "" LSAPGPU_FILTER_RB=1 > $O/sweep_c4.txt 2>&1
for t in 8 16 32; do LSAPGPU_UPLOAD_THREADS=$t timeout 300 python tools/e2e_probe.py >> $O/e2e_threads.txt 2>&1; done
