"""Full-sweep duration from the device timeline (first scan stamp -> next stamp)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1106_5694_b200 as g
ctx = g.Context(0)
ctx.generate(sys.argv[1] if len(sys.argv) > 1 else "p2p", int(sys.argv[2]) if len(sys.argv) > 2 else 10000, 0)
ctx.set_timeline(1 << 12)
out = []
for _ in range(6):
    ctx.timeline()
    ctx.solve(g.ParallelConfig(seed=0), trace=False)
    tl = ctx.timeline()
    t1 = next((t for t, k in tl if k == 1), None)
    t3 = next((t for t, k in tl if k == 3 and t1 is not None and t > t1), None)
    if t1 is not None and t3 is not None:
        out.append((t3 - t1) / 1e3)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
print(os.environ.get("LSAPGPU_SCAN_L2PF", "-"), "full sweep us:", [round(x, 1) for x in out],
      "GB/s(int16):", round(2 * n * n * 2 / (min(out[1:]) * 1e-6) / 1e9))
