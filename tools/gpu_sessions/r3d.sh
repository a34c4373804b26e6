O=gpurun_out/r3d; mkdir -p $O
for pf in 0 4096; do echo "pf=$pf" >> $O/e2e.txt; LSAPGPU_HOST_TIMING=1 LSAPGPU_NARROW_PF=$pf timeout 300 python tools/e2e_probe.py 2>&1 | grep -E "upload timing|e2e ms" | tail -3 >> $O/e2e.txt; done
python tools/h2d_bench.py > $O/h2d.txt 2>&1
