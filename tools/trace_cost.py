"""Where the objective trace's cost goes in a C3 solve: host marks of the
library (LSAPGPU_HOST_TIMING, printed to stderr per solve) for trace on / off,
and the Python wrapper's share (event-timed solve minus the library's own
elapsed).

    LSAPGPU_HOST_TIMING=1 python tools/trace_cost.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1106_5694_b200 as g

ctx = g.Context(0)
ctx.generate("p2p", 10000, 0)
cfg = g.ParallelConfig(seed=0)
for trace in (True, False, True, False):
    ts, el = [], []
    for _ in range(8):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = ctx.solve(cfg, trace=trace)
        ts.append((time.perf_counter() - t0) * 1e3)
        el.append(r.elapsed / 1e6)
    sys.stderr.flush()
    print(f"trace={trace}: wall {np.median(ts[2:]):.3f} ms, library elapsed {np.median(el[2:]):.3f} ms", flush=True)
