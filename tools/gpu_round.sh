#!/bin/bash
# One GPU session: tests, smoke, bench, launch list, ncu --set full of the pair scan.
# Usage (from the repo root, under gpurun): bash tools/gpu_round.sh [tag]
TAG=${1:-r1}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file $O/launches.csv python tools/profile_target.py > $O/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_scan -s 0 -c 3 \
  -o $O/pair_scan python tools/profile_target.py > $O/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:commit -s 5 -c 1 \
  -o $O/commit python tools/profile_target.py > $O/ncu_commit.log 2>&1
ls -la $O
