"""Determinism matrix of the long-row scan: objective of repeated solves vs the
streaming kernel under env variants.  python tools/c5_matrix.py n [VAR=v,...] ..."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json; sys.path.insert(0, %r)
import paper_1106_5694_b200 as g
n = %d
ctx = g.Context(0); ctx.generate("f32", n, 0)
res = []
for k in range(4):
    r = ctx.solve(g.ParallelConfig(seed=0, use_graph=(k %% 2 == 0)))
    res.append([r.assignment.value, r.gpu["inner_iterations"], r.switches_applied, r.gpu["filter_overflows"]])
print(json.dumps({"plan": ctx.scan_plan(), "solves": res}))
'''
n = int(sys.argv[1])
for spec in sys.argv[2:]:
    env = dict(os.environ)
    for kv in filter(None, spec.split(",")):
        k, v = kv.split("="); env[k] = v
    r = subprocess.run([sys.executable, "-c", CHILD % (ROOT, n)], env=env, capture_output=True, text=True, timeout=1200)
    line = [l for l in r.stdout.splitlines() if l.startswith("{")]
    print(n, spec or "default", line[-1] if line else r.stderr[-800:], flush=True)
