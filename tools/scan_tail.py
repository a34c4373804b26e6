"""Per-CTA completion spread of every scan launch (deep device timeline)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1106_5694_b200 as g
ctx = g.Context(0)
ctx.generate(sys.argv[1] if len(sys.argv) > 1 else "p2p", int(sys.argv[2]) if len(sys.argv) > 2 else 10000, 0)
ctx.set_timeline(1 << 15)
ctx.solve(g.ParallelConfig(seed=0), trace=False)
ctx.timeline()
r = ctx.solve(g.ParallelConfig(seed=0), trace=False)
tl = ctx.timeline(1 << 15)
t0 = tl[0][0]
cur = None
rows = []
for t, k in tl:
    if k in (1, 2):
        cur = {"start": t, "ends": [], "multi": 0, "kind": k}
        rows.append(cur)
    elif k in (11, 12) and cur is not None:
        cur["ends"].append(t)
        cur["multi"] += k == 12
    elif k == 3 and cur is not None:
        cur["next"] = t
for r_ in rows:
    e = sorted(r_["ends"])
    if not e:
        continue
    nxt = r_.get("next", e[-1])
    print(f"scan@{(r_['start'] - t0) / 1e3:8.1f}  ctas {len(e):3d} multi {r_['multi']:3d}  first_end {(e[0] - r_['start']) / 1e3:6.2f}"
          f"  median_end {(e[len(e) // 2] - r_['start']) / 1e3:6.2f}  last_end {(e[-1] - r_['start']) / 1e3:6.2f}"
          f"  next_kernel {(nxt - r_['start']) / 1e3:6.2f} us")
