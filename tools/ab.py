"""A/B solve timing across plan variants (fresh process per variant).

    python tools/ab.py '[{}, {"LSAPGPU_SCAN_SEGMENTS": "4"}]' [kind n solves]

Prints min / median graph-mode solve time (SolveReport.elapsed) per variant,
variants interleaved over rounds to average out box drift."""
import json, os, subprocess, sys, statistics
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, json; sys.path.insert(0, %r)
import paper_1106_5694_b200 as g
ctx = g.Context(0); ctx.generate(%r, %d, 0)
ts = []
for _ in range(%d):
    r = ctx.solve(g.ParallelConfig(seed=0), trace=False); ts.append(r.elapsed / 1e3)
print(json.dumps(ts[1:]))
'''
variants = json.loads(sys.argv[1])
kind = sys.argv[2] if len(sys.argv) > 2 else "p2p"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 10000
solves = int(sys.argv[4]) if len(sys.argv) > 4 else 8
res = {i: [] for i in range(len(variants))}
for rnd in range(3):
    for i, env in enumerate(variants):
        e = dict(os.environ, **env)
        r = subprocess.run([sys.executable, "-c", code % (ROOT, kind, n, solves)], env=e, capture_output=True, text=True)
        try:
            res[i] += json.loads(r.stdout.strip().splitlines()[-1])
        except Exception:
            print(env, r.stderr[-600:])
for i, env in enumerate(variants):
    v = res[i]
    if v:
        print(f"{json.dumps(env):60s} min {min(v):8.1f} us  median {statistics.median(v):8.1f} us  (n={len(v)})")
