O=gpurun_out/r4j; mkdir -p $O
lscpu | grep -E "Model name|^CPU\(s\)|NUMA" > $O/lscpu.txt 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 python bench.py > $O/bench2.json 2> $O/bench2.err
