O=gpurun_out/r4c; mkdir -p $O
echo "## tools/fuzz_parity.py 4000 41 (default plans, round-2 final code)" >> $O/fuzz.txt
timeout 1500 python tools/fuzz_parity.py 4000 41 2>&1 | tail -2 >> $O/fuzz.txt
echo "## LSAPGPU_SCAN_FILTER=2 tools/fuzz_parity.py 1500 43 (filter scan, aux in TMEM)" >> $O/fuzz.txt
LSAPGPU_SCAN_FILTER=2 timeout 1500 python tools/fuzz_parity.py 1500 43 2>&1 | tail -2 >> $O/fuzz.txt
echo "## LSAPGPU_SCAN_FILTER=2 LSAPGPU_FILTER_BITS=8 tools/fuzz_parity.py 1000 47 (int8 copies, aux in TMEM)" >> $O/fuzz.txt
LSAPGPU_SCAN_FILTER=2 LSAPGPU_FILTER_BITS=8 timeout 1500 python tools/fuzz_parity.py 1000 47 2>&1 | tail -2 >> $O/fuzz.txt
S="compute-sanitizer --tool memcheck --print-limit 5"
(echo "## memcheck host-stepped, LSAPGPU_SCAN_FILTER=2 (aux in TMEM)"; LSAPGPU_SCAN_FILTER=2 timeout 1200 $S python tools/dgs_sanitize.py 2>&1 | grep -E "ERROR SUMMARY" | head -3) >> $O/sanitizer.txt
(echo "## synccheck host-stepped, LSAPGPU_SCAN_FILTER=2 (aux in TMEM)"; LSAPGPU_SCAN_FILTER=2 timeout 1200 compute-sanitizer --tool synccheck python tools/dgs_sanitize.py 2>&1 | grep -E "ERROR SUMMARY" | head -3) >> $O/sanitizer.txt
