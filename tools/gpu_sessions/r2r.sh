O=gpurun_out/r2r; mkdir -p $O
lscpu > $O/lscpu.txt 2>&1; free -g >> $O/lscpu.txt 2>&1
for t in 16; do LSAPGPU_UPLOAD_THREADS=$t timeout 300 python tools/e2e_probe.py >> $O/e2e_threads.txt 2>&1; done
timeout 600 python tools/timeline.py --solves 2 > $O/timeline_c3.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_scan_res -s 2 -c 1 -o $O/res_c3_reeval python tools/profile_target.py --stepped > $O/ncu_res.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_scan_res -s 0 -c 1 -o $O/res_c3_full python tools/profile_target.py --stepped > $O/ncu_res_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:commit_cluster -s 0 -c 1 -o $O/commit_c3 python tools/profile_target.py --stepped > $O/ncu_commit.log 2>&1
timeout 900 python tools/filter_sweep.py c4 "" LSAPGPU_FILTER_WARPS=24 > $O/sweep_c4.txt 2>&1
