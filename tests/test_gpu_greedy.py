"""Greedy initial assignment (extension, BASELINE north star item 2; not in
the reference, whose dgs_parallel always starts from initial_random): the
device rule against the oracle's restatement, and DGS solves from the greedy
start against the oracle's dgs loop from the same start (bit-exact)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = [("int", 1000, 3, 1000.0), ("int", 3000, 4, 100000.0), ("p2p", 2000, 5, None), ("f32", 1500, 6, None),
         ("unit", 800, 7, 10.0), ("geom", 700, 8, 100.0), ("int", 257, 9, 7.0)]


@pytest.mark.parametrize("kind,n,seed,param", CASES)
def test_greedy_assignment_matches_oracle(oracle, gpu_ctx, kind, n, seed, param):
    a = oracle.generate(kind, n, seed, param)
    gpu_ctx.set_matrix(a)
    sigma, rounds = gpu_ctx.greedy_assignment()
    want, wrounds = oracle.greedy_assignment(a)
    assert np.array_equal(sigma, want)
    assert rounds == wrounds


@pytest.mark.parametrize("kind,n,seed,param", CASES)
@pytest.mark.parametrize("graph", [True, False])
def test_solve_from_greedy_start(oracle, gpu_ctx, kind, n, seed, param, graph):
    import paper_1106_5694_b200 as g
    a = oracle.generate(kind, n, seed, param)
    gpu_ctx.set_matrix(a)
    rep = gpu_ctx.solve(g.ParallelConfig(init="greedy", use_graph=graph))
    start, _ = oracle.greedy_assignment(a)
    want = oracle.dgs_parallel_from(a, start)
    assert np.array_equal(rep.assignment.sigma, want.sigma)
    assert rep.assignment.value == want.value
    assert rep.outer_iterations == want.outer_iterations
    assert rep.switches_applied == want.switches_applied
    assert rep.objective_trace == want.trace


def test_greedy_start_on_device_generated_c3(oracle, gpu_ctx):
    """C3 (n=10k P2P) from the greedy start, sigma vs the oracle loop."""
    import paper_1106_5694_b200 as g
    gpu_ctx.generate("p2p", 10000, 0)
    rep = gpu_ctx.solve(g.ParallelConfig(init="greedy"), trace=False)
    a = oracle.generate("p2p", 10000, 0)
    start, _ = oracle.greedy_assignment(a)
    want = oracle.dgs_parallel_from(a, start, trace=False)
    assert np.array_equal(rep.assignment.sigma, want.sigma)
    assert rep.assignment.value == want.value
