"""set_matrix from pageable host fp64 (the drop-in C++ Instance path): ms per call.
    LSAPGPU_UPLOAD_THREADS=k python tools/pageable_probe.py [n]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1106_5694_b200 as g
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
a = g.generate_instance("p2p", n, 0)
ctx = g.Context(0)
ts = []
for _ in range(6):
    t0 = time.perf_counter()
    ctx.set_matrix(a)
    ts.append((time.perf_counter() - t0) * 1e3)
print(os.environ.get("LSAPGPU_UPLOAD_THREADS", "default"), "threads: pageable set_matrix ms",
      [round(t, 2) for t in ts], "cpus", os.cpu_count(), flush=True)
