"""Per-batch phase table of one graph-mode C3 solve from the device timeline:
for every inner batch, the scan (launch -> first stage -> CTA 0 done), the
gap to the commit, the commit and the apply, in microseconds.

    python tools/timeline_batches.py [--kind p2p --n 10000]"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1106_5694_b200 as g

ap = argparse.ArgumentParser()
ap.add_argument("--kind", default="p2p"); ap.add_argument("--n", type=int, default=10000)
a = ap.parse_args()
ctx = g.Context(0)
ctx.generate(a.kind, a.n, 0)
ctx.set_timeline(8192)
ctx.solve(g.ParallelConfig(seed=0))
ctx.timeline()
r = ctx.solve(g.ParallelConfig(seed=0))
tl = ctx.timeline()
t0 = tl[0][0]
ev = [((t - t0) / 1e3, k) for t, k in tl]
# kinds: 1 full_sweep, 2 scan, 3 commit:start, 4 commit:end, 8 res:acur, 9 res:stage0, 10 res:cta0_done, 15 apply
rows, cur = [], {}
for t, k in ev:
    if k in (1, 2):
        if cur:
            rows.append(cur)
        cur = {"scan": t, "full": k == 1}
    elif k == 9 and "stage0" not in cur:
        cur["stage0"] = t
    elif k == 10:
        cur["cta0"] = t
    elif k == 3:
        cur["cstart"] = t
    elif k == 4:
        cur["cend"] = t
    elif k == 15:
        cur["apply"] = t
if cur:
    rows.append(cur)
print(f"solve elapsed {r.elapsed / 1e3:.1f} us, {len(rows)} scans")
print("  #  kind  prologue   scan  ->commit  commit  ->apply  apply->next")
tot = {"pro": 0.0, "scan": 0.0, "gap": 0.0, "commit": 0.0, "ga": 0.0, "an": 0.0}
for i, c in enumerate(rows):
    nxt = rows[i + 1]["scan"] if i + 1 < len(rows) else None
    pro = c.get("stage0", c["scan"]) - c["scan"]
    sc = c.get("cta0", c.get("stage0", c["scan"])) - c.get("stage0", c["scan"])
    gap = c["cstart"] - c.get("cta0", c["scan"]) if "cstart" in c else 0.0
    com = c["cend"] - c["cstart"] if "cend" in c and "cstart" in c else 0.0
    ga = c["apply"] - c["cend"] if "apply" in c and "cend" in c else 0.0
    an = nxt - c["apply"] if nxt is not None and "apply" in c else 0.0
    for k, v in zip(tot, (pro, sc, gap, com, ga, an)):
        tot[k] += v
    print(f"{i:3d}  {'full' if c['full'] else 'list':4s}  {pro:7.1f} {sc:7.1f}  {gap:7.1f} {com:7.1f}  {ga:7.1f}  {an:7.1f}")
print("sum  " + "  ".join(f"{k} {v:.1f}" for k, v in tot.items()))
