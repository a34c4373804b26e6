O=gpurun_out/r3r; mkdir -p $O
for w in c1 c2; do timeout 900 python bench.py --workload $w > $O/bench_$w.json 2> $O/bench_$w.err; done
for w in c4 c5; do timeout 1500 python bench.py --workload $w --no-cpu --steps 5 > $O/bench_$w.json 2> $O/bench_$w.err; done
