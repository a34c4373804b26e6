"""Minimal ncu target: one C3 solve (or --kind/--n) through the C-ABI.
--src host uploads the oracle-generated fp64 matrix (the bench path);
--src device builds it with the on-device generator."""
import argparse, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1106_5694_b200 as g
ap = argparse.ArgumentParser()
ap.add_argument("--kind", default="p2p"); ap.add_argument("--n", type=int, default=10000)
ap.add_argument("--stepped", action="store_true"); ap.add_argument("--solves", type=int, default=1)
ap.add_argument("--src", default="device", choices=["device", "host", "devfp64"])
ap.add_argument("--trace", action="store_true", help="objective trace on (the bench's setting)")
a = ap.parse_args()
ctx = g.Context(0)
if a.src == "host":
    from oracle.oracle import Oracle
    ctx.set_matrix(Oracle().generate(a.kind, a.n, 0))
elif a.src == "devfp64":  # the bench's value step: fp64 matrix in HBM -> set_matrix (layout) -> solve
    import torch
    ctx.set_matrix(torch.from_numpy(g.generate_instance(a.kind, a.n, 0)).cuda())
else:
    ctx.generate(a.kind, a.n, 0)
for _ in range(a.solves):
    r = ctx.solve(g.ParallelConfig(seed=0, use_graph=not a.stepped), trace=a.trace)
print(r.assignment.value, r.gpu)
