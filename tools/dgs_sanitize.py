"""Small host-stepped solves for compute-sanitizer (memcheck / racecheck):
resident and streaming scans, both commits, greedy start, step APIs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1106_5694_b200 as g
ctx = g.Context(0)
for kind, n, param in [("int", 700, 1000.0), ("p2p", 900, None), ("geom", 300, 100.0), ("f32", 500, None)]:
    ctx.generate(kind, n, 1, param)
    for init in ("random", "greedy"):
        for pol in ("touched_and_conflicted", "touched_only"):
            r = ctx.solve(g.ParallelConfig(seed=2, use_graph=False, init=init, reeval=pol))
            print(kind, n, init, pol, r.assignment.value, flush=True)
    sig, rounds = ctx.greedy_assignment()
    t = ctx.evaluate_all(sig)
    print("step apis ok", len(ctx.check_conflicts(t, sig).reserved), flush=True)
