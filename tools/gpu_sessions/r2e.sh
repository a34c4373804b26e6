O=gpurun_out/r2e; mkdir -p $O
export LSAPGPU_SCAN_FILTER=2
timeout 600 compute-sanitizer --tool memcheck --show-backtrace no python tools/filter_debug.py 1000 > $O/memcheck_1000.txt 2>&1
unset LSAPGPU_SCAN_FILTER
timeout 900 python -m pytest tests/test_gpu_filter.py -x -q > $O/pytest_filter.log 2>&1; echo "rc=$?" >> $O/pytest_filter.log
timeout 900 python -m pytest tests/test_gpu_golden.py -x -q > $O/pytest_golden.log 2>&1; echo "rc=$?" >> $O/pytest_golden.log
timeout 600 python bench.py --workload c4 --no-cpu --steps 3 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err
timeout 600 python bench.py --workload c5 --no-cpu --steps 2 --warmup 2 > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_scan -s 0 -c 1 -o $O/filter_c4_full python tools/profile_target.py --kind f32 --n 30000 --stepped > $O/ncu_c4.log 2>&1
