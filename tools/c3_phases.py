"""Split the C3 bench step (device fp64 -> layout -> solve -> sigma/tau on host)
into its host-visible phases, CUDA-event timed on the context's stream.

    python tools/c3_phases.py [--n 10000] [--reps 10]"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1106_5694_b200 as g

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=10000); ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
ctx = g.Context(0)
a_dev = torch.from_numpy(g.generate_instance("p2p", a.n, 0)).cuda()
strm = torch.cuda.ExternalStream(ctx.stream)
cfg = g.ParallelConfig(seed=0)


def timed(f):
    ts = []
    for _ in range(a.reps + 3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(strm); r = f(); e1.record(strm); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts[3:])), r


t_set, _ = timed(lambda: ctx.set_matrix(a_dev))
t_solve_tr, r = timed(lambda: ctx.solve(cfg))
t_solve_nt, r2 = timed(lambda: ctx.solve(cfg, trace=False))
t_step, _ = timed(lambda: (ctx.set_matrix(a_dev), ctx.solve(cfg)))
print(f"set_matrix(device fp64) {t_set:.3f} ms")
print(f"solve trace on          {t_solve_tr:.3f} ms   (report elapsed {r.elapsed / 1e6:.3f} ms)")
print(f"solve trace off         {t_solve_nt:.3f} ms")
print(f"step (bench value)      {t_step:.3f} ms")
print("gpu stats:", {k: r.gpu[k] for k in ("inner_iterations", "pair_items", "launches") if k in r.gpu})
