O=gpurun_out/r2g; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 ./build/cpp/test_lsapgpu > $O/cpp_test.log 2>&1; echo "rc=$?" >> $O/cpp_test.log
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_scan -s 0 -c 1 -o $O/filter_c4_full python tools/profile_target.py --kind f32 --n 30000 --stepped > $O/ncu_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_scan -s 0 -c 1 -o $O/filter_c5_full python tools/profile_target.py --kind f32 --n 100000 --stepped > $O/ncu_c5.log 2>&1
