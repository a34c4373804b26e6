O=gpurun_out/r3u; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_deadline.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for r in 1 2; do timeout 300 python tools/timeline_batches.py 2>&1 | grep -E "^sum|elapsed" >> $O/timeline.txt; timeout 300 python tools/c3_phases.py 2>&1 | grep -E "solve trace on|step" >> $O/timeline.txt; done
