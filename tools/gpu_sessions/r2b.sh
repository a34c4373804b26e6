O=gpurun_out/r2b; mkdir -p $O
timeout 300 ./tools/micro/tma_rate > $O/tma_rate.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_deadline.py -x -q > $O/pytest_deadline.log 2>&1; echo "rc=$?" >> $O/pytest_deadline.log
