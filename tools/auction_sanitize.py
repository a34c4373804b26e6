"""Small auction runs for compute-sanitizer (memcheck / racecheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1106_5694_b200 as g
ctx = g.Context(0)
for kind, n, seed, param, cfg in [("int", 300, 1, 1000.0, {}), ("geom", 128, 2, 100.0, {"scaling": True}),
                                   ("geom", 200, 3, 100.0, {"deadline": 0}), ("p2p", 500, 4, None, {})]:
    ctx.generate(kind, n, seed, param)
    r = ctx.auction_solve(g.AuctionConfig(**cfg))
    print(kind, n, r.outer_iterations, r.assignment.value, flush=True)
os.environ["LSAPGPU_AUCTION_LOCAL_PRICES"] = "0"
ctx.generate("int", 300, 1, 1000.0)
print("global prices", ctx.auction_solve(g.AuctionConfig()).outer_iterations)
