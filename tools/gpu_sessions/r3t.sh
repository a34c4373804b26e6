O=gpurun_out/r3t; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_upload.py tests/test_gpu_golden.py tests/test_gpu_dist.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for r in 1 2; do timeout 300 python tools/c3_phases.py >> $O/phases.txt 2>&1; done
P="python tools/profile_target.py --src devfp64 --trace --stepped"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:layout_ -s 1 -c 1 -o $O/layout $P > $O/ncu_layout.log 2>&1
