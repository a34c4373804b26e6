import sys, time
sys.path.insert(0, '.')
import paper_1106_5694_b200 as g
from oracle.oracle import Oracle
o = Oracle()
ctx = g.Context(0)
for kind, n in [("int", 1000), ("p2p", 10000), ("f32", 10000)]:
    t = time.time(); ctx.generate(kind, n, 0); t1 = time.time() - t
    for ug in (True, False):
        t = time.time(); r = ctx.solve(g.ParallelConfig(seed=0, use_graph=ug), trace=False); t2 = time.time() - t
        print(kind, n, "graph" if ug else "stepped", "gen %.1fms solve %.1fms" % (t1*1e3, t2*1e3), r.assignment.value, r.gpu, flush=True)
# per-phase timing (host-stepped, CUDA events around every scan / commit launch)
for kind, n in [("p2p", 10000), ("f32", 10000)]:
    ctx.generate(kind, n, 0)
    ctx.set_scan_timing(True)
    r = ctx.solve(g.ParallelConfig(seed=0, use_graph=False))
    ctx.set_scan_timing(False)
    tm = ctx.scan_timing()
    print(kind, n, "phases", tm, "bytes", r.gpu["bytes_scanned"],
          "scan GB/s %.0f" % (r.gpu["bytes_scanned"] / tm["scan_ms"] / 1e6),
          "full GB/s %.0f" % (2 * n * n * ctx.storage_bytes * tm["full_launches"] / tm["full_ms"] / 1e6), flush=True)
