O=gpurun_out/r3l; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_upload.py tests/test_gpu_golden.py tests/test_gpu_filter.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for r in 1 2; do timeout 300 python tools/c3_phases.py >> $O/phases.txt 2>&1; done
P="python tools/profile_target.py --src devfp64 --trace --stepped"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:layout_fused -s 1 -c 1 -o $O/layout $P > $O/ncu_layout.log 2>&1
for r in 1 2; do
  for v in 0 4; do echo "## variant $v" >> $O/timeline_ab.txt; LSAPGPU_COMMIT_VARIANT=$v timeout 300 python tools/timeline_batches.py 2>&1 | grep -E "^sum|elapsed" >> $O/timeline_ab.txt; done
done
LSAPGPU_COMMIT_VARIANT=4 timeout 1800 python -m pytest tests/test_gpu_golden.py -x -q > $O/pytest_variant4.log 2>&1; echo "rc=$?" >> $O/pytest_variant4.log
