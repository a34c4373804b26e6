O=gpurun_out/r4i; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 3000 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 ./build/cpp/test_lsapgpu > $O/cpp_test.log 2>&1; echo "rc=$?" >> $O/cpp_test.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
P="python tools/profile_target.py --src devfp64 --trace --stepped"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_scan_res -s 0 -c 2 -o $O/pair_scan $P > $O/ncu_scan.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches_c3_stepped.csv $P > $O/launches.log 2>&1
timeout 300 python tools/timeline_batches.py > $O/timeline_batches.txt 2>&1
