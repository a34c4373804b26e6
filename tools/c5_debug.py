"""C5 determinism probe: evaluate_all tables and repeated solves under the current env plan."""
import hashlib, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1106_5694_b200 as g
n = int(sys.argv[1]); tag = sys.argv[2]
ctx = g.Context(0); ctx.generate("f32", n, 0)
s = g.random_perm(n, 4)
t = ctx.evaluate_all(s)
h = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]
out = {"tag": tag, "plan": ctx.scan_plan(), "tables": [h(t.agent_delta), h(t.agent_partner), h(t.job_delta), h(t.job_partner)]}
np.save(f"gpurun_out/c5dbg_{tag}_{n}.npy", np.stack([t.agent_delta, t.agent_partner.astype(np.float64), t.job_delta, t.job_partner.astype(np.float64)]))
objs = []
for k in range(3):
    r = ctx.solve(g.ParallelConfig(seed=0, use_graph=(k != 2)))
    objs.append((r.assignment.value, r.gpu["inner_iterations"], r.switches_applied))
out["solves"] = objs
print(json.dumps(out), flush=True)
