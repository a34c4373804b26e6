#!/bin/bash
# Stepped launch list + ncu captures of re-eval scans and commit kernels, H2D probe.
TAG=${1:-probe}
O=gpurun_out/$TAG
mkdir -p $O
timeout 300 python tools/h2d_bench.py > $O/h2d.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file $O/launches_stepped.csv python tools/profile_target.py --stepped > $O/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_scan -s 2 -c 3 \
  -o $O/pair_scan_reeval python tools/profile_target.py --stepped > $O/ncu_reeval.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:commit -s 3 -c 2 \
  -o $O/commit python tools/profile_target.py --stepped > $O/ncu_commit.log 2>&1
ls -la $O
