O=gpurun_out/r3z; mkdir -p $O
for r in 1 2; do
  for v in 0 1; do
    for c in c4 c5; do echo "TMEM=$v $(timeout 900 python tools/filter_sweep.py $c LSAPGPU_FILTER_TMEM=$v 2>&1 | tail -1)" >> $O/tmem_ab.txt; done
  done
done
timeout 3000 python -m pytest tests/test_gpu_filter.py -x -q > $O/pytest_filter.log 2>&1; echo "rc=$?" >> $O/pytest_filter.log
