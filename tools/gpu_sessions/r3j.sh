O=gpurun_out/r3j; mkdir -p $O
for r in 1 2; do
  for v in 8 16; do echo "V=$v $(timeout 600 python tools/filter_sweep.py c5 LSAPGPU_FILTER_V=$v 2>&1 | tail -1)" >> $O/filter_v.txt; done
done
timeout 2400 python -m pytest tests/test_gpu_filter.py -x -q > $O/pytest_filter.log 2>&1; echo "rc=$?" >> $O/pytest_filter.log
(cd tools/micro && ./graph_rebuild_memcheck && compute-sanitizer --tool memcheck --print-limit 2 ./graph_rebuild_memcheck && compute-sanitizer --tool memcheck --print-limit 2 ./graph_rebuild_memcheck cluster) > $O/graph_rebuild_memcheck.txt 2>&1
P="python tools/profile_target.py --src devfp64 --trace --stepped"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:layout_fused -s 1 -c 1 -o $O/layout $P > $O/ncu_layout.log 2>&1
