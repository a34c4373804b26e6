O=gpurun_out/r4b; mkdir -p $O
for r in 1 2; do
  echo "default $(timeout 900 python tools/filter_sweep.py c5 2>&1 | tail -1)" >> $O/c5_ab.txt
  echo "rb2q512 $(timeout 900 python tools/filter_sweep.py c5 LSAPGPU_FILTER_RB=2,LSAPGPU_FILTER_QUEUE=512 2>&1 | tail -1)" >> $O/c5_ab.txt
done
