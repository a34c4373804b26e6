"""Randomised parity sweep: device solves vs the oracle restatement, bit for bit.

    python tools/fuzz_parity.py [count] [seed]

Random kind / n / instance seed / solver seed / policy / eps / graph mode /
init mode; prints every mismatch and a summary line."""
import os, random, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1106_5694_b200 as g
from oracle.oracle import Oracle

count = int(sys.argv[1]) if len(sys.argv) > 1 else 100
rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
o = Oracle()
ctx = g.Context(0)
bad = 0
t0 = time.time()
for k in range(count):
    kind = rng.choice(["int", "int", "unit", "geom", "f32", "p2p", "intbig", "neg"])
    n = rng.choice([2, 3, 5, 17, 64, 65, 127, 300, 513, 1000, 1500, 2048, 3000])
    iseed, sseed = rng.randrange(1 << 30), rng.randrange(1 << 30)
    if kind == "intbig":
        a = o.generate("int", n, iseed, 1 << 20)
    elif kind == "neg":
        a = o.generate("int", n, iseed, 200.0) - 100.0
    else:
        a = o.generate(kind, n, iseed, {"int": 1000.0, "unit": 10.0, "geom": 100.0}.get(kind))
    policy = rng.choice(["touched_and_conflicted", "touched_and_conflicted", "touched_only"])
    eps = rng.choice([0.0, 0.0, 0.0, 0.5, 2.0])
    graph = rng.choice([True, True, False])
    init = rng.choice(["random", "random", "greedy"])
    ctx.set_matrix(a)
    rep = ctx.solve(g.ParallelConfig(seed=sseed, reeval=policy, improvement_epsilon=eps, use_graph=graph,
                                     init=init))
    pol = 0 if policy == "touched_and_conflicted" else 1
    if init == "greedy":
        start, _ = o.greedy_assignment(a)
        want = o.dgs_parallel_from(a, start, eps=eps, policy=pol)
    else:
        want = o.dgs_parallel(a, seed=sseed, eps=eps, policy=pol)
    ok = (np.array_equal(rep.assignment.sigma, want.sigma) and rep.assignment.value == want.value and
          rep.outer_iterations == want.outer_iterations and rep.switches_applied == want.switches_applied and
          rep.objective_trace == want.trace)
    if not ok:
        bad += 1
        print(f"MISMATCH {kind} n={n} iseed={iseed} seed={sseed} {policy} eps={eps} graph={graph} init={init}: "
              f"value {rep.assignment.value} vs {want.value}, switches {rep.switches_applied} vs "
              f"{want.switches_applied}", flush=True)
print(f"fuzz: {count} solves, {bad} mismatches, {time.time() - t0:.0f} s", flush=True)
sys.exit(1 if bad else 0)
