O=gpurun_out/r2p; mkdir -p $O
timeout 1200 python tools/filter_sweep.py c4 "" LSAPGPU_FILTER_FLAGS=1 "" LSAPGPU_FILTER_FLAGS=1 > $O/sweep_c4.txt 2>&1
timeout 1200 python tools/filter_sweep.py c5 "" LSAPGPU_FILTER_FLAGS=1 LSAPGPU_FILTER_RB=1 LSAPGPU_FILTER_RB=1,LSAPGPU_FILTER_FLAGS=1 > $O/sweep_c5.txt 2>&1
