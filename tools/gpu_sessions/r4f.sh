O=gpurun_out/r4f; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_upload.py tests/test_gpu_filter.py -x -q -k "upload or misspec or bit_exact" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for r in 1 2 3; do
  LSAPGPU_HOST_TIMING=1 timeout 300 python tools/e2e_probe.py 2>&1 | grep -E "upload timing|e2e ms" | tail -2 >> $O/e2e.txt
  (cd scratch/ab_base && LSAPGPU_HOST_TIMING=1 timeout 300 python tools/e2e_probe.py 2>&1 | grep -E "upload timing|e2e ms" | tail -2 | sed 's/^/base /') >> $O/e2e.txt
done
