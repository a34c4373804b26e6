O=gpurun_out/r3b; mkdir -p $O
g++ -O2 -mavx2 -pthread tools/micro/host_read.cpp -o tools/micro/host_read
for pf in 0 512 1024 2048 4096; do echo "PF=$pf" >> $O/host_read.txt; LSAPGPU_NARROW_PF=$pf ./tools/micro/host_read 10000 2>&1 | grep -E "threads (8|12|16) " >> $O/host_read.txt; done
for pf in 0 1024 2048; do echo "pf=$pf $(LSAPGPU_NARROW_PF=$pf timeout 300 python tools/e2e_probe.py 2>&1 | tail -1)" >> $O/e2e.txt; done
for pf in 0 1024 2048; do echo "pf=$pf $(LSAPGPU_NARROW_PF=$pf timeout 300 python tools/e2e_probe.py 2>&1 | tail -1)" >> $O/e2e.txt; done
