"""Graph-mode phase breakdown of one solve from the device timeline.

    python tools/timeline.py [--kind p2p --n 10000] [--solves 3]

Each scan / commit launch stamps %globaltimer at entry (CTA 0); a phase's
duration is the gap to the next stamp, so launch gaps count toward the phase
they precede.  Commit end stamps split the commit from the following gap."""
import argparse, collections, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1106_5694_b200 as g

ap = argparse.ArgumentParser()
ap.add_argument("--kind", default="p2p"); ap.add_argument("--n", type=int, default=10000)
ap.add_argument("--solves", type=int, default=3)
a = ap.parse_args()
ctx = g.Context(0)
ctx.generate(a.kind, a.n, 0)
ctx.set_timeline(8192)
names = {1: "full_sweep", 2: "scan", 3: "commit:start", 4: "commit:end", 5: "single:loaded",
         6: "single:round_end", 7: "res:tau16", 8: "res:acur", 9: "res:stage0", 10: "res:cta0_done",
         11: "cl:P1done", 12: "cl:round_end", 13: "cl:phaseA", 14: "cl:classified", 15: "apply"}
for k in range(a.solves):
    ctx.timeline()  # clear
    r = ctx.solve(g.ParallelConfig(seed=0), trace=False)
    tl = ctx.timeline()
    agg = collections.defaultdict(lambda: [0, 0.0])
    for (t0, kind), (t1, _) in zip(tl, tl[1:]):
        agg[names[kind]][0] += 1
        agg[names[kind]][1] += (t1 - t0) / 1e3
    span = (tl[-1][0] - tl[0][0]) / 1e3 if tl else 0
    print(f"solve {k}: elapsed {r.elapsed/1e3:.1f} us, first->last stamp {span:.1f} us, "
          f"inner {r.gpu['inner_iterations']}, items {r.gpu['pair_items']}")
    for nm, (c, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"   {nm:14s} {c:4d}  {us:9.1f} us  avg {us / max(c, 1):7.2f} us")
# raw sequence of the last solve's final iterations
if tl:
    t0 = tl[0][0]
    print("raw tail:", [(round((t - t0) / 1e3, 2), names.get(k, k)) for t, k in tl[:80]])
# resolution check
ts = sorted(t for t, _ in tl)
d = [b - a for a, b in zip(ts, ts[1:]) if b > a]
print("min stamp gap ns:", min(d) if d else None)
