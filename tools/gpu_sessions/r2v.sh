O=gpurun_out/r2v; mkdir -p $O
g++ -O2 -mavx2 -pthread tools/micro/host_read.cpp -o tools/micro/host_read && ./tools/micro/host_read > $O/host_read.txt 2>&1
lscpu > $O/lscpu.txt 2>&1
for r in 1 2; do
  for v in base cur; do
    if [ $v = base ]; then D=scratch/ab_base; else D=.; fi
    echo "== $v round $r" >> $O/phases.txt
    (cd $D && timeout 300 python tools/c3_phases.py) >> $O/phases.txt 2>&1
    (cd $D && timeout 300 python tools/e2e_probe.py) >> $O/phases.txt 2>&1
  done
done
timeout 300 python tools/timeline.py --solves 2 > $O/timeline_cur.txt 2>&1
(cd scratch/ab_base && timeout 300 python tools/timeline.py --solves 2) > $O/timeline_base.txt 2>&1
