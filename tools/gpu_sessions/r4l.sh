O=gpurun_out/r4l; mkdir -p $O
for r in 1 2 3; do
  for cfg in "1 32" "0 8" "0 4" "1 8"; do set -- $cfg
    echo "nt=$1 mb=$2 $(LSAPGPU_NARROW_NT=$1 LSAPGPU_NARROW_CHUNK_MB=$2 timeout 300 python tools/e2e_probe.py 2>&1 | tail -1)" >> $O/e2e_ab.txt
  done
done
