O=gpurun_out/r3g; mkdir -p $O
# filter kernel A/B: rotated aux register sets (working tree) vs HEAD
for r in 1 2; do
  for c in c4 c5; do
    echo "cur $c $(timeout 600 python tools/filter_sweep.py $c 2>&1 | tail -1)" >> $O/filter_ab.txt
    echo "base $c $(cd scratch/ab_base && timeout 600 python tools/filter_sweep.py $c 2>&1 | tail -1)" >> $O/filter_ab.txt
  done
done
timeout 1200 python -m pytest tests/test_gpu_filter.py -x -q > $O/pytest_filter.log 2>&1; echo "rc=$?" >> $O/pytest_filter.log
# memcheck graph-mode false-positive check
LSAPGPU_PDL=0 timeout 1200 compute-sanitizer --tool memcheck python tools/dgs_sanitize.py graph > $O/memcheck_graph_nopdl.log 2>&1; echo "rc=$?" >> $O/memcheck_graph_nopdl.log
