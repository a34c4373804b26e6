"""One or two solves for a targeted compute-sanitizer run.
    python tools/sanitize_min.py kind n init[,init2] graph(0|1) [policy]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1106_5694_b200 as g
kind, n, inits, graph = sys.argv[1], int(sys.argv[2]), sys.argv[3].split(","), sys.argv[4] == "1"
pol = sys.argv[5] if len(sys.argv) > 5 else "touched_and_conflicted"
ctx = g.Context(0)
ctx.generate(kind, n, 1, {"int": 1000.0, "geom": 100.0}.get(kind))
for init in inits:
    if init == "greedy_only":  # the greedy kernel alone (cooperative launch), no solve
        ctx.greedy_assignment()
        print("greedy_assignment", flush=True)
        continue
    r = ctx.solve(g.ParallelConfig(seed=2, use_graph=graph, init=init, reeval=pol))
    print(kind, n, init, "graph" if graph else "stepped", r.assignment.value, flush=True)
