O=gpurun_out/r3i; mkdir -p $O
S="compute-sanitizer --tool memcheck --print-limit 2"
run() { name=$1; shift; echo "## $name: $*" >> $O/min.txt; timeout 900 "$@" > $O/$name.log 2>&1; echo "rc=$?" >> $O/min.txt; grep -E "ERROR SUMMARY|^int|^geom|^p2p|^greedy|Invalid|  at " $O/$name.log | head -8 >> $O/min.txt; }
run f_geom_random_greedyonly_random $S python tools/sanitize_min.py geom 300 random,greedy_only,random 1
run g_int_random_greedyonly_random $S python tools/sanitize_min.py int 700 random,greedy_only,random 1
SANITIZE_INITS=random run h_full_random_graph $S python tools/dgs_sanitize.py graph
SANITIZE_INITS=random LSAPGPU_SCAN_FILTER=2 run i_full_random_graph_filter $S python tools/dgs_sanitize.py graph
bash tools/gpu_sessions/r3f.sh
