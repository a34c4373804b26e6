O=gpurun_out/r3x; mkdir -p $O
P="python tools/profile_target.py --kind f32 --n 30000 --stepped"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pair_scan_filter -s 0 -c 2 -o $O/filter_c4 $P > $O/ncu_c4.log 2>&1
timeout 900 python tools/big_timing.py > $O/big_timing.txt 2>&1
