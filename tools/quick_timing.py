import sys, time, numpy as np
sys.path.insert(0, '.')
import paper_1106_5694_b200 as g
from oracle.oracle import Oracle
o = Oracle()
ctx = g.Context(0)
for kind, n in [("int", 1000), ("p2p", 10000), ("f32", 10000)]:
    t = time.time(); ctx.generate(kind, n, 0); t1 = time.time() - t
    for ug in (True, False):
        t = time.time(); r = ctx.solve(g.ParallelConfig(seed=0, use_graph=ug)); t2 = time.time() - t
        print(kind, n, "graph" if ug else "stepped", "gen %.1fms solve %.1fms" % (t1*1e3, t2*1e3), r.assignment.value, r.gpu, flush=True)
