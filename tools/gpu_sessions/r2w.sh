O=gpurun_out/r2w; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_upload.py tests/test_gpu_parity.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for r in 1 2; do
  for t in 16 12 14; do
    LSAPGPU_UPLOAD_THREADS=$t timeout 300 python tools/e2e_probe.py >> $O/e2e.txt 2>&1
  done
  (cd scratch/ab_base && timeout 300 python tools/e2e_probe.py) | sed 's/^/base /' >> $O/e2e.txt 2>&1
done
