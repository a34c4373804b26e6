O=gpurun_out/r2x; mkdir -p $O
LSAPGPU_HOST_TIMING=1 timeout 300 python tools/e2e_probe.py > $O/e2e_timing.txt 2>&1
LSAPGPU_HOST_TIMING=1 timeout 300 python tools/trace_cost.py > $O/trace_cost.txt 2>&1
