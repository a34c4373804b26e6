"""Solve time from the greedy start vs the reference's random start (device).

    python tools/greedy_timing.py [kind n]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1106_5694_b200 as g
kind = sys.argv[1] if len(sys.argv) > 1 else "p2p"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
ctx = g.Context(0)
ctx.generate(kind, n, 0, 1000.0 if kind == "int" else None)
for init in ("random", "greedy"):
    ts = []
    for _ in range(6):
        r = ctx.solve(g.ParallelConfig(init=init), trace=False)
        ts.append(r.elapsed / 1e3)
    print(f"{kind} n={n} init={init:6s} solve min {min(ts[1:]):8.1f} us  value {r.assignment.value!r} "
          f"switches {r.switches_applied} inner {r.gpu['inner_iterations']} outer {r.outer_iterations}", flush=True)
sig, rounds = ctx.greedy_assignment()
print("greedy rounds", rounds)
