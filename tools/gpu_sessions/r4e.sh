O=gpurun_out/r4e; mkdir -p $O
for r in 1 2 3; do
  echo "cur $(timeout 900 python tools/filter_sweep.py c4 2>&1 | tail -1)" >> $O/c4_ab.txt
  echo "base $(cd scratch/ab_base && timeout 900 python tools/filter_sweep.py c4 2>&1 | tail -1)" >> $O/c4_ab.txt
done
timeout 3000 python -m pytest tests/test_gpu_filter.py -x -q > $O/pytest_filter.log 2>&1; echo "rc=$?" >> $O/pytest_filter.log
