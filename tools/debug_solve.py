import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1106_5694_b200 as g
from oracle.oracle import Oracle
o = Oracle()
kind = sys.argv[1] if len(sys.argv) > 1 else "int"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 300
graph = (sys.argv[3] == "graph") if len(sys.argv) > 3 else False
a = o.generate(kind, n, 11)
ctx = g.Context(0)
ctx.set_matrix(a)
r = ctx.solve(g.ParallelConfig(seed=2, use_graph=graph))
q = o.dgs_parallel(a, seed=2)
print("match", np.array_equal(r.assignment.sigma, q.sigma), r.objective_trace == q.trace, r.gpu)
