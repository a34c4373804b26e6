"""Randomised auction parity sweep: device vs the oracle restatement.

    python tools/fuzz_auction.py [count] [seed]"""
import os, random, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1106_5694_b200 as g
from oracle.oracle import Oracle

count = int(sys.argv[1]) if len(sys.argv) > 1 else 100
rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
o = Oracle()
ctx = g.Context(0)
bad = 0
t0 = time.time()
for k in range(count):
    kind = rng.choice(["int", "unit", "geom", "f32", "p2p", "neg"])
    n = rng.choice([1, 2, 3, 7, 33, 100, 257, 500, 800])
    iseed = rng.randrange(1 << 30)
    if kind == "neg":
        a = o.generate("int", n, iseed, 60.0) - 30.0
    else:
        a = o.generate(kind, n, iseed, {"int": rng.choice([5.0, 1000.0]), "unit": 10.0, "geom": 100.0}.get(kind))
    cfg = {}
    r = rng.random()
    if r < 0.3:
        cfg["epsilon"] = rng.choice([0.01, 0.3, 1.0, 0.9 / max(n, 1)])
    if rng.random() < 0.4:
        cfg["scaling"] = True
        cfg["scale_factor"] = rng.choice([2.0, 4.0, 7.5])
    ctx.set_matrix(a)
    rep = ctx.auction_solve(g.AuctionConfig(**cfg))
    want = o.auction_solve(a, **cfg)
    ok = (np.array_equal(rep.assignment.sigma, want.sigma) and rep.assignment.value == want.value and
          rep.outer_iterations == want.rounds and rep.switches_applied == want.switches and
          np.array_equal(rep.gpu["prices"].view(np.int64), want.prices.view(np.int64)))
    if not ok:
        bad += 1
        print(f"MISMATCH {kind} n={n} iseed={iseed} cfg={cfg}: rounds {rep.outer_iterations} vs {want.rounds}",
              flush=True)
print(f"auction fuzz: {count} solves, {bad} mismatches, {time.time() - t0:.0f} s", flush=True)
sys.exit(1 if bad else 0)
