O=gpurun_out/r4g; mkdir -p $O
timeout 1500 python tools/ab.py '[{}, {"LSAPGPU_SCAN_M": "1", "LSAPGPU_SCAN_BUFS": "4"}, {"LSAPGPU_SCAN_M": "1", "LSAPGPU_SCAN_BUFS": "3"}, {"LSAPGPU_SCAN_L2PF": "1"}]' p2p 10000 8 > $O/ab_res.txt 2>&1
