O=gpurun_out/r2d; mkdir -p $O
export LSAPGPU_SCAN_FILTER=2
timeout 600 compute-sanitizer --tool memcheck --show-backtrace no python tools/filter_debug.py 1000 > $O/memcheck_1000.txt 2>&1
timeout 600 compute-sanitizer --tool memcheck --show-backtrace no python tools/filter_debug.py 10000 > $O/memcheck_10000.txt 2>&1
unset LSAPGPU_SCAN_FILTER
timeout 900 python -m pytest tests/test_gpu_upload.py -x -q > $O/pytest_upload.log 2>&1; echo "rc=$?" >> $O/pytest_upload.log
