O=gpurun_out; 
for n in 100000 60000; do
python tools/c5_debug.py $n rb2 > $O/c5dbg_rb2_$n.txt 2>&1
LSAPGPU_FILTER_RB=1 python tools/c5_debug.py $n rb1 > $O/c5dbg_rb1_$n.txt 2>&1
LSAPGPU_SCAN_FILTER=0 python tools/c5_debug.py $n stream > $O/c5dbg_stream_$n.txt 2>&1
done
python -c "
import numpy as np
for n in (100000, 60000):
    a=np.load('gpurun_out/c5dbg_rb2_%d.npy'%n); b=np.load('gpurun_out/c5dbg_rb1_%d.npy'%n); c=np.load('gpurun_out/c5dbg_stream_%d.npy'%n)
    for nm,x in (('rb2',a),('rb1',b)):
        d=(x!=c); print(n, nm, 'mismatch rows', d.sum(axis=1), 'first', [np.nonzero(r)[0][:5].tolist() for r in d])
" > $O/c5dbg_cmp.txt 2>&1
rm -f gpurun_out/c5dbg_*.npy
