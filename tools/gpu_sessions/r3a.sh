O=gpurun_out/r3a; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_golden.py tests/test_gpu_parity.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
LSAPGPU_HOST_TIMING=1 timeout 300 python tools/trace_cost.py > $O/trace_cost.txt 2>&1
timeout 300 python tools/c3_phases.py > $O/phases.txt 2>&1
timeout 300 python tools/e2e_probe.py > $O/e2e.txt 2>&1
