"""C3 drop-in e2e (pageable fp64 Instance -> lsap.dgs_parallel) under the current env."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1106_5694_b200 as g
a = g.generate_instance("p2p", 10000, 0).copy()
inst = g.Instance(10000, a)
cfg = g.ParallelConfig(seed=0)
ctx = g.context(0)
for _ in range(3):
    g.dgs_parallel(inst, cfg)
ts = []
for _ in range(8):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    g.dgs_parallel(inst, cfg)
    torch.cuda.synchronize(); ts.append((time.perf_counter() - t0) * 1e3)
t_up = []
for _ in range(5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    ctx.set_instance(inst); torch.cuda.synchronize(); t_up.append((time.perf_counter() - t0) * 1e3)
print("threads", os.environ.get("LSAPGPU_UPLOAD_THREADS"), "e2e ms", round(float(np.median(ts)), 2), "upload ms", round(float(np.median(t_up)), 2), "cpus", os.cpu_count())
