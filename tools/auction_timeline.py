"""Per-phase breakdown of auction rounds from the device timeline (CTA 0).

    python tools/auction_timeline.py [case]"""
import collections, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1106_5694_b200 as g
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
nm = sys.argv[1] if len(sys.argv) > 1 else "c2_int5000"
rec = json.load(open(os.path.join(ROOT, "tests", "golden", "auction.json")))["cases"][nm]
ctx = g.Context(0)
ctx.generate(rec["kind"], rec["n"], rec["instance_seed"], rec["param"])
ctx.set_timeline(1 << 16)
names = {1: "top->bid_done", 2: "bid_done->sync1", 3: "apply", 4: "apply_done->sync2/top"}
for _ in range(2):
    ctx.timeline()
    r = ctx.auction_solve(g.AuctionConfig())
    tl = ctx.timeline(1 << 16)
agg = collections.defaultdict(lambda: [0, 0.0])
for (t0, k0), (t1, _) in zip(tl, tl[1:]):
    agg[names[k0]][0] += 1
    agg[names[k0]][1] += (t1 - t0) / 1e3
print(nm, "rounds", r.outer_iterations, "elapsed ms", r.elapsed / 1e6, "stamps", len(tl))
for k, (c, us) in agg.items():
    print(f"  {k:24s} {c:6d} {us:10.1f} us  avg {us / max(c, 1):6.2f} us")
