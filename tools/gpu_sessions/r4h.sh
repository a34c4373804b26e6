O=gpurun_out/r4h; mkdir -p $O
timeout 1500 python tools/ab.py '[{}, {"LSAPGPU_SCAN_L2PF": "1"}, {"LSAPGPU_SCAN_L2PF": "2"}, {"LSAPGPU_SCAN_L2PF": "4"}]' p2p 10000 8 > $O/ab_pf_c3.txt 2>&1
timeout 1500 python tools/ab.py '[{}, {"LSAPGPU_SCAN_L2PF": "1"}, {"LSAPGPU_SCAN_L2PF": "2"}]' int 5000 8 > $O/ab_pf_c2.txt 2>&1
timeout 1500 python tools/ab.py '[{}, {"LSAPGPU_SCAN_L2PF": "1"}]' int 1000 8 > $O/ab_pf_c1.txt 2>&1
