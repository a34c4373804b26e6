"""Scan-tail breakdown from deep timeline stamps (per-CTA end marks, tl cap > 8192).

    python tools/scan_tail2.py [kind n]

Per scan launch: CTA-0 done, first / median / last CTA end, next commit start."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1106_5694_b200 as g
kind = sys.argv[1] if len(sys.argv) > 1 else "p2p"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
ctx = g.Context(0)
ctx.generate(kind, n, 0)
ctx.set_timeline(1 << 17)
for _ in range(2):
    ctx.timeline(1 << 17)
    r = ctx.solve(g.ParallelConfig(seed=0), trace=False)
    tl = ctx.timeline(1 << 17)
rows = []
cur = None
for t, k in tl:
    if k in (1, 2):
        cur = {"start": t, "ends": [], "cta0": None}
    elif cur is not None and k == 10:
        cur["cta0"] = t
    elif cur is not None and k in (11, 12) and cur.get("commit") is None:
        cur["ends"].append(t)
    elif cur is not None and k == 3 and cur.get("commit") is None:
        cur["commit"] = t
        rows.append(cur)
        cur = None
print(f"{'#':>3} {'scan':>7} {'cta0':>7} {'first':>7} {'med':>7} {'last':>7} {'commit':>7}  (us from scan start)")
tails, launch = [], []
for q, rw in enumerate(rows):
    s0 = rw["start"]
    e = sorted(rw["ends"]) or [s0]
    f = lambda t: (t - s0) / 1e3 if t else float("nan")
    if q < 40:
        print(f"{q:3d} {len(e):7d} {f(rw['cta0']):7.1f} {f(e[0]):7.1f} {f(e[len(e)//2]):7.1f} {f(e[-1]):7.1f} {f(rw['commit']):7.1f}")
    tails.append((e[-1] - (rw["cta0"] or e[-1])) / 1e3)
    launch.append((rw["commit"] - e[-1]) / 1e3)
print("avg last_end - cta0 %.2f us, avg commit_start - last_end %.2f us over %d scans" %
      (statistics.mean(tails), statistics.mean(launch), len(rows)))
