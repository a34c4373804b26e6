O=gpurun_out/r3h; mkdir -p $O
S="compute-sanitizer --tool memcheck --print-limit 2"
run() { name=$1; shift; echo "## $name: $*" >> $O/min.txt; timeout 600 "$@" > $O/$name.log 2>&1; echo "rc=$?" >> $O/min.txt; grep -E "ERROR SUMMARY|^int|^geom|^p2p|Invalid|  at " $O/$name.log | head -8 >> $O/min.txt; }
run a_int_graph_pdl $S python tools/sanitize_min.py int 700 random 1
LSAPGPU_PDL=0 run b_geom_greedy_graph_nopdl $S python tools/sanitize_min.py geom 300 greedy 1
LSAPGPU_PDL=0 run c_geom_random_greedy_graph_nopdl $S python tools/sanitize_min.py geom 300 random,greedy 1
LSAPGPU_PDL=0 run d_geom_random_graph_nopdl $S python tools/sanitize_min.py geom 300 random,random 1
run e_int_stepped_pdl $S python tools/sanitize_min.py int 700 random 0
