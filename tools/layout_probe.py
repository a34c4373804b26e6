"""Time set_matrix from a device-resident fp64 matrix (the bench 'value' layout phase)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1106_5694_b200 as g
kind = sys.argv[1] if len(sys.argv) > 1 else "p2p"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
a = torch.from_numpy(g.generate_instance(kind, n, 0)).cuda()
ctx = g.Context(0)
s = torch.cuda.ExternalStream(ctx.stream)
ts = []
for _ in range(8):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    ctx.set_matrix(a)
    e1.record(s)
    e1.synchronize()
    ts.append(e0.elapsed_time(e1))
print("set_matrix(device fp64) ms:", [round(t, 3) for t in ts])
