O=gpurun_out/r3v; mkdir -p $O
timeout 1500 python tools/ab.py '[{}, {"LSAPGPU_COMMIT_CS": "8"}, {"LSAPGPU_COMMIT_SINGLE_MAX": "2048"}, {"LSAPGPU_COMMIT_SINGLE": "0"}]' p2p 10000 8 > $O/ab_commit.txt 2>&1
