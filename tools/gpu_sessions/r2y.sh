O=gpurun_out/r2y; mkdir -p $O
for nt in 1 0; do for mb in 8 16 32 64; do
  echo "nt=$nt mb=$mb $(LSAPGPU_NARROW_NT=$nt LSAPGPU_NARROW_CHUNK_MB=$mb timeout 300 python tools/e2e_probe.py 2>&1 | tail -1)" >> $O/sweep.txt
done; done
for nt in 1 0; do for mb in 16 32; do
  echo "nt=$nt mb=$mb $(LSAPGPU_NARROW_NT=$nt LSAPGPU_NARROW_CHUNK_MB=$mb timeout 300 python tools/e2e_probe.py 2>&1 | tail -1)" >> $O/sweep.txt
done; done
LSAPGPU_HOST_TIMING=1 timeout 300 python tools/trace_cost.py > $O/trace_cost.txt 2>&1
