O=gpurun_out/r3w; mkdir -p $O
LSAPGPU_FILTER_TMEM=1 timeout 600 python tools/filter_sweep.py c4 > $O/smoke_tmem.txt 2>&1; echo "rc=$?" >> $O/smoke_tmem.txt
for r in 1 2; do
  for v in 0 1; do echo "TMEM=$v $(timeout 600 python tools/filter_sweep.py c4 LSAPGPU_FILTER_TMEM=$v 2>&1 | tail -1)" >> $O/tmem_ab.txt; done
done
timeout 2400 python -m pytest tests/test_gpu_filter.py -x -q > $O/pytest_filter.log 2>&1; echo "rc=$?" >> $O/pytest_filter.log
