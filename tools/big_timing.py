"""Timing of the large configs (C4 30k fp32, C5 100k fp32) on one GPU."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1106_5694_b200 as g
ctx = g.Context(0)
for kind, n in [(a.split(":")[0], int(a.split(":")[1])) for a in (sys.argv[1:] or ["f32:30000", "f32:100000"])]:
    t = time.time(); ctx.generate(kind, n, 0); tg = time.time() - t
    for rep in range(2):
        t = time.time(); r = ctx.solve(g.ParallelConfig(seed=0), trace=False); ts = time.time() - t
        print(kind, n, "gen %.0fms solve %.1fms" % (tg * 1e3, ts * 1e3), r.assignment.value, r.gpu, flush=True)
    ctx.set_scan_timing(True)
    r = ctx.solve(g.ParallelConfig(seed=0, use_graph=False), trace=False)
    ctx.set_scan_timing(False)
    tm = ctx.scan_timing()
    print(kind, n, "phases", tm, "scan GB/s %.0f" % (r.gpu["bytes_scanned"] / tm["scan_ms"] / 1e6),
          "full GB/s %.0f" % (2 * n * n * ctx.storage_bytes * tm["full_launches"] / tm["full_ms"] / 1e6), flush=True)
