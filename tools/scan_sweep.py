"""Sweep scan plans (M items per CTA stage, B staged buffers) in fresh processes."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, json; sys.path.insert(0, %r)
import paper_1106_5694_b200 as g
ctx = g.Context(0)
out = {}
for kind, n in %s:
    ctx.generate(kind, n, 0)
    ctx.solve(g.ParallelConfig(seed=0, use_graph=False))
    ctx.set_scan_timing(True)
    r = ctx.solve(g.ParallelConfig(seed=0, use_graph=False))
    ctx.set_scan_timing(False)
    tm = ctx.scan_timing()
    eb = ctx.storage_bytes
    out[f"{kind}{n}"] = dict(full_gbs=round(2*n*n*eb*tm["full_launches"]/tm["full_ms"]/1e6),
                             scan_gbs=round(r.gpu["bytes_scanned"]/tm["scan_ms"]/1e6),
                             scan_ms=round(tm["scan_ms"],3), commit_ms=round(tm["commit_ms"],3),
                             solve_ms=round(r.elapsed/1e6,3))
print(json.dumps(out))
'''
cases = sys.argv[1] if len(sys.argv) > 1 else "[('p2p', 10000), ('f32', 10000)]"
grid = [(256, 4, 1, 2), (256, 4, 1, 3), (256, 2, 1, 3), (256, 2, 2, 2), (256, 2, 2, 3), (256, 2, 2, 4),
        (256, 4, 2, 2), (256, 4, 2, 3), (256, 1, 2, 3), (256, 1, 2, 4)]
if len(sys.argv) > 2:
    grid = json.loads(sys.argv[2])
for nt, m, b, dd in grid:
    env = dict(os.environ, LSAPGPU_SCAN_M=str(m), LSAPGPU_SCAN_BUFS=str(b), LSAPGPU_SCAN_NT=str(nt),
               LSAPGPU_SCAN_DEPTH=str(dd))
    r = subprocess.run([sys.executable, "-c", code % (ROOT, cases)], env=env, capture_output=True, text=True)
    print(f"NT={nt} M={m} B={b} D={dd}", r.stdout.strip() or r.stderr[-500:], flush=True)
