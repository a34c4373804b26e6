O=gpurun_out/r3k; mkdir -p $O
echo "## tools/fuzz_parity.py 3000 23 (default plans)" >> $O/fuzz.txt
timeout 1500 python tools/fuzz_parity.py 3000 23 2>&1 | tail -3 >> $O/fuzz.txt; echo "rc=$?" >> $O/fuzz.txt
echo "## LSAPGPU_SCAN_FILTER=2 tools/fuzz_parity.py 1000 29 (quantized-filter scan at every n, int16 copies)" >> $O/fuzz.txt
LSAPGPU_SCAN_FILTER=2 timeout 1500 python tools/fuzz_parity.py 1000 29 2>&1 | tail -3 >> $O/fuzz.txt; echo "rc=$?" >> $O/fuzz.txt
echo "## LSAPGPU_SCAN_FILTER=2 LSAPGPU_FILTER_BITS=8 tools/fuzz_parity.py 1000 31 (int8 copies)" >> $O/fuzz.txt
LSAPGPU_SCAN_FILTER=2 LSAPGPU_FILTER_BITS=8 timeout 1500 python tools/fuzz_parity.py 1000 31 2>&1 | tail -3 >> $O/fuzz.txt; echo "rc=$?" >> $O/fuzz.txt
echo "## LSAPGPU_SCAN_RESIDENT=0 LSAPGPU_SCAN_FILTER=0 tools/fuzz_parity.py 500 37 (streaming scan)" >> $O/fuzz.txt
LSAPGPU_SCAN_RESIDENT=0 LSAPGPU_SCAN_FILTER=0 timeout 1500 python tools/fuzz_parity.py 500 37 2>&1 | tail -3 >> $O/fuzz.txt; echo "rc=$?" >> $O/fuzz.txt
S="compute-sanitizer --tool memcheck --print-limit 5"
(echo "## memcheck host-stepped, default plans"; timeout 1200 $S python tools/dgs_sanitize.py 2>&1 | grep -E "ERROR SUMMARY|^upload|Error" | head -8) >> $O/sanitizer.txt
(echo "## memcheck host-stepped, LSAPGPU_SCAN_FILTER=2"; LSAPGPU_SCAN_FILTER=2 timeout 1200 $S python tools/dgs_sanitize.py 2>&1 | grep -E "ERROR SUMMARY|^upload|Error" | head -8) >> $O/sanitizer.txt
(echo "## synccheck host-stepped, LSAPGPU_SCAN_FILTER=2"; LSAPGPU_SCAN_FILTER=2 timeout 1200 compute-sanitizer --tool synccheck python tools/dgs_sanitize.py 2>&1 | grep -E "ERROR SUMMARY" | head -3) >> $O/sanitizer.txt
(echo "## memcheck graph mode, fresh graph (random start): tools/sanitize_min.py int 700 random 1 / p2p 900 random,random 1"; timeout 600 $S python tools/sanitize_min.py int 700 random 1 2>&1 | grep -E "ERROR SUMMARY"; timeout 600 $S python tools/sanitize_min.py p2p 900 random,random 1 2>&1 | grep -E "ERROR SUMMARY"; LSAPGPU_SCAN_FILTER=2 timeout 600 $S python tools/sanitize_min.py f32 1500 random,random 1 2>&1 | grep -E "ERROR SUMMARY") >> $O/sanitizer.txt
