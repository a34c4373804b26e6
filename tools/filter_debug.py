"""Small filter-kernel case for compute-sanitizer: evaluate_all vs the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1106_5694_b200 as g
from oracle.oracle import Oracle
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
o = Oracle(); ctx = g.Context(0)
a = o.generate("f32", n, 11)
ctx.set_matrix(a)
print(ctx.scan_plan(), flush=True)
s = o.random_perm(n, 4)
t = ctx.evaluate_all(s)
ad, ap, jd, jp = o.evaluate_all(a, s)
print("agent ok", np.array_equal(t.agent_partner, ap), np.array_equal(t.agent_delta, ad))
print("job ok", np.array_equal(t.job_partner, jp), np.array_equal(t.job_delta, jd))
r = ctx.solve(g.ParallelConfig(seed=2, use_graph=False)); q = o.dgs_parallel(a, seed=2)
print("solve ok", np.array_equal(r.assignment.sigma, q.sigma))
