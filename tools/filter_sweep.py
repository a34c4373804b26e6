"""Full-sweep timing of the long-row scan at C4 / C5 under plan variants
(each variant in a fresh process: the plan is read from the environment when
the matrix is set).  python tools/filter_sweep.py [c4|c5] VAR=val,VAR=val ..."""
import json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json; sys.path.insert(0, %r)
import paper_1106_5694_b200 as g
n = %d
ctx = g.Context(0); ctx.generate("f32", n, 0)
ctx.solve(g.ParallelConfig(seed=0))  # warm: first touch of every buffer, graph build
ctx.set_scan_timing(True)
r = ctx.solve(g.ParallelConfig(seed=0, use_graph=False))
ctx.set_scan_timing(False)
tm = ctx.scan_timing()
t0 = __import__("time").time()
r2 = ctx.solve(g.ParallelConfig(seed=0))
print(json.dumps({"plan": ctx.scan_plan(), "full_ms": tm["full_ms"] / max(tm["full_launches"], 1),
                  "scan_ms": tm["scan_ms"], "solve_ms": r2.elapsed / 1e6, "kept_per_item": r.gpu["filter_kept"] / r.gpu["pair_items"],
                  "overflows": r.gpu["filter_overflows"], "objective": r.assignment.value}))
'''
wl = sys.argv[1] if len(sys.argv) > 1 else "c4"
n = {"c4": 30000, "c5": 100000}[wl]
for spec in sys.argv[2:] or [""]:
    env = dict(os.environ)
    for kv in filter(None, spec.split(",")):
        k, v = kv.split("=")
        env[k] = v
    r = subprocess.run([sys.executable, "-c", CHILD % (ROOT, n)], env=env, capture_output=True, text=True, timeout=900)
    line = [l for l in r.stdout.splitlines() if l.startswith("{")]
    print(wl, spec or "default", line[-1] if line else r.stderr[-500:], flush=True)
