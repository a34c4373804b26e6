"""CTA 0 stage trace of the first full sweep (deep device timeline):
P = producer got the buffer, S0 = warp 0 starts the stage, SL = last consumer warp
starts, R = the stage's last warp releases the buffer."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1106_5694_b200 as g
ctx = g.Context(0)
ctx.generate(sys.argv[1] if len(sys.argv) > 1 else "p2p", int(sys.argv[2]) if len(sys.argv) > 2 else 10000, 0)
ctx.set_timeline(1 << 15)
ctx.solve(g.ParallelConfig(seed=0), trace=False)
ctx.timeline()
ctx.solve(g.ParallelConfig(seed=0), trace=False)
tl = ctx.timeline(1 << 15)
t0 = tl[0][0]
end = next(t for t, k in tl if k == 3)
ev = sorted((t, k) for t, k in tl if t < end and k in (11, 12, 13, 14))
name = {11: "S0", 12: "R", 13: "P", 14: "SL"}
line = []
for t, k in ev[:160]:
    line.append(f"{name[k]}@{(t - t0) / 1e3:.2f}")
print(" ".join(line))
