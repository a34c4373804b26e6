O=gpurun_out/r3e; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_upload.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
g++ -O2 -mavx2 -pthread tools/micro/host_read.cpp -o tools/micro/host_read
for pf in 4096 8192; do echo "PF=$pf" >> $O/host_read.txt; LSAPGPU_NARROW_PF=$pf ./tools/micro/host_read 10000 2>&1 | grep -E "threads (12|16) " >> $O/host_read.txt; done
for r in 1 2 3; do LSAPGPU_HOST_TIMING=1 timeout 300 python tools/e2e_probe.py 2>&1 | grep -E "upload timing|e2e ms" | tail -2 >> $O/e2e.txt; done
bash tools/gpu_sessions/r3c.sh
