"""Small solves for compute-sanitizer (memcheck / racecheck / synccheck):
resident, streaming and filter scans (whichever the environment's plan
selects), both commits, both policies, greedy start, graph and host-stepped
passes, the device log ordering (trace on), the host-narrowed upload and the
step APIs.

    compute-sanitizer --tool memcheck python tools/dgs_sanitize.py [graph]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1106_5694_b200 as g

graph_modes = (False, True) if (len(sys.argv) > 1 and sys.argv[1] == "graph") else (False,)
ctx = g.Context(0)
for kind, n, param in [("int", 700, 1000.0), ("p2p", 900, None), ("geom", 300, 100.0), ("f32", 500, None)]:
    ctx.generate(kind, n, 1, param)
    for use_graph in graph_modes:
        for init in os.environ.get("SANITIZE_INITS", "random,greedy").split(","):
            for pol in ("touched_and_conflicted", "touched_only"):
                r = ctx.solve(g.ParallelConfig(seed=2, use_graph=use_graph, init=init, reeval=pol))
                print(kind, n, "graph" if use_graph else "stepped", init, pol, r.assignment.value,
                      len(r.objective_trace), r.gpu["host_log_orders"], flush=True)
    sig, rounds = ctx.greedy_assignment()
    t = ctx.evaluate_all(sig)
    print("step apis ok", len(ctx.check_conflicts(t, sig).reserved), flush=True)
# host upload with host-side narrowing (int16 / fp32 speculation, fp64 fallback)
rng = np.random.default_rng(0)
for a in (rng.integers(0, 3000, (600, 600)).astype(np.float64),
          rng.random((500, 500)).astype(np.float32).astype(np.float64),
          rng.random((400, 400))):
    ctx.set_matrix(a)
    r = ctx.solve(g.ParallelConfig(seed=1, use_graph=graph_modes[-1]))
    print("upload", a.shape[0], ctx.scan_plan()["kernel"], r.assignment.value, flush=True)
