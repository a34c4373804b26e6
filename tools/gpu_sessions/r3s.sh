O=gpurun_out/r3s; mkdir -p $O
timeout 1200 python tools/ab.py '[{}, {"LSAPGPU_SCAN_RES_NT": "640"}, {"LSAPGPU_SCAN_RES_NT": "768"}]' p2p 10000 8 > $O/ab_nt.txt 2>&1
timeout 900 python tools/ab.py '[{}, {"LSAPGPU_SCAN_RES_NT": "640"}, {"LSAPGPU_SCAN_RES_NT": "768"}]' int 5000 8 > $O/ab_nt_c2.txt 2>&1
