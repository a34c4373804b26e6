O=gpurun_out/r4k; mkdir -p $O
timeout 1800 python tools/ab.py '[{}, {"LSAPGPU_SCAN_SEGMENTS": "2"}, {"LSAPGPU_SCAN_SEGMENTS": "4"}, {"LSAPGPU_APPLY_CTAS": "32"}, {"LSAPGPU_APPLY_CTAS": "128"}]' p2p 10000 8 > $O/ab_misc.txt 2>&1
