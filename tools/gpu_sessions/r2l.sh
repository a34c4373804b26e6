O=gpurun_out/r2l; mkdir -p $O
timeout 1500 python tools/c5_matrix.py 100000 LSAPGPU_FILTER_CHECK=1 LSAPGPU_FILTER_CHECK=1,LSAPGPU_FILTER_RB=1 "" > $O/check.txt 2>&1
timeout 900 python tools/c5_matrix.py 60000 LSAPGPU_FILTER_CHECK=1,LSAPGPU_FILTER_BITS=8 LSAPGPU_FILTER_BITS=8 >> $O/check.txt 2>&1
timeout 900 python tools/c5_matrix.py 30000 "" >> $O/check.txt 2>&1
