O=gpurun_out/r2n; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_filter.py tests/test_gpu_golden.py tests/test_gpu_upload.py -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python bench.py --workload c1 --no-cpu --steps 3 > $O/bench_blocks.json 2> $O/bench_blocks.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_c4.csv python tools/profile_target.py --kind f32 --n 30000 --stepped > $O/launches_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_scan_filter -s 0 -c 1 -o $O/filter_c4_full python tools/profile_target.py --kind f32 --n 30000 --stepped > $O/ncu_c4.log 2>&1
