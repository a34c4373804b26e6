O=gpurun_out/r2q; mkdir -p $O
timeout 1500 python tools/filter_sweep.py c4 "" LSAPGPU_FILTER_WARPS=24 "" LSAPGPU_FILTER_WARPS=24 > $O/sweep_c4.txt 2>&1
timeout 1500 python tools/filter_sweep.py c5 "" LSAPGPU_FILTER_WARPS=24 > $O/sweep_c5.txt 2>&1
timeout 900 python tools/c5_matrix.py 100000 LSAPGPU_FILTER_WARPS=24,LSAPGPU_FILTER_CHECK=5 > $O/check.txt 2>&1
