O=gpurun_out/r3f; mkdir -p $O
P="python tools/profile_target.py --src devfp64 --trace --stepped"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $O/launches_c3_stepped.csv $P > $O/launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:layout_fused -c 1 -o $O/layout $P > $O/ncu_layout.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:order_log -c 1 -o $O/order_log $P > $O/ncu_order.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_scan_res -s 0 -c 3 -o $O/pair_scan $P > $O/ncu_scan.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:commit_cluster -s 0 -c 1 -o $O/commit $P > $O/ncu_commit.log 2>&1
timeout 300 python tools/timeline_batches.py > $O/timeline_batches.txt 2>&1
timeout 600 python tools/big_timing.py > $O/big_timing.txt 2>&1
ls -la $O
