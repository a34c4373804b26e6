O=gpurun_out/r2a; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 300 ./tools/micro/l2_rate > $O/l2_rate.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py --workload c4 --no-cpu --steps 3 --warmup 3 > $O/bench_c4.json 2> $O/bench_c4.err
