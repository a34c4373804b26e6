O=gpurun_out/r3c; mkdir -p $O
S=compute-sanitizer
run() { name=$1; shift; echo "## $name" >> $O/sanitizer.txt; timeout 1200 "$@" > $O/$name.log 2>&1; echo "rc=$?" >> $O/sanitizer.txt; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Program hit|Invalid" $O/$name.log | sort | uniq -c | head -5 >> $O/sanitizer.txt; }
run memcheck_graph $S --tool memcheck python tools/dgs_sanitize.py graph
LSAPGPU_SCAN_FILTER=2 run memcheck_filter_graph $S --tool memcheck python tools/dgs_sanitize.py graph
LSAPGPU_SCAN_RESIDENT=0 run memcheck_streaming $S --tool memcheck python tools/dgs_sanitize.py
run racecheck_stepped $S --tool racecheck python tools/dgs_sanitize.py
LSAPGPU_SCAN_FILTER=2 run racecheck_filter $S --tool racecheck python tools/dgs_sanitize.py
run synccheck_stepped $S --tool synccheck python tools/dgs_sanitize.py
