O=gpurun_out/r2h; mkdir -p $O
timeout 900 python tools/filter_sweep.py c4 "" LSAPGPU_FILTER_BITS=8 LSAPGPU_FILTER_BITS=8,LSAPGPU_FILTER_RB=1 LSAPGPU_FILTER_RB=1 > $O/sweep_c4.txt 2>&1
timeout 900 python tools/filter_sweep.py c5 "" LSAPGPU_FILTER_RB=1 > $O/sweep_c5.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
