O=gpurun_out/r4a; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 3000 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 ./build/cpp/test_lsapgpu > $O/cpp_test.log 2>&1; echo "rc=$?" >> $O/cpp_test.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
for w in c4 c5; do timeout 1500 python bench.py --workload $w --no-cpu --steps 5 > $O/bench_$w.json 2> $O/bench_$w.err; done
P="python tools/profile_target.py --kind f32 --stepped"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_scan_filter -s 0 -c 2 -o $O/filter_c4 $P --n 30000 > $O/ncu_c4.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:pair_scan_filter -s 0 -c 1 -o $O/filter_c5 $P --n 100000 > $O/ncu_c5.log 2>&1
