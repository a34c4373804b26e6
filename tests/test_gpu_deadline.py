"""GPU: the anytime deadline fires on the device, mid-pass.

The reference checks its Deadline every 16 scans and after every batch
(parallel.cpp:91,114,336; solver_state.hpp:13-27).  The device checks
%globaltimer at the end of every batch's commit; the host only checks at pass
boundaries.  Each case below cuts a solve inside its FIRST pass (outer
iteration 1, fewer batches than the full solve), which only the device check
can do, and checks what the reference guarantees of an anytime result: a
permutation, value == the ordered objective of that permutation
(snapshot_assignment, solver_state.hpp:141-148), a non-decreasing trace and
terminated_by == deadline.  Multi-rank solves must agree on the batch at which
they stop (the deadline vote travels with the record exchange, dist.cu)."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def ordered_objective(a, sigma):
    v = 0.0
    for j, i in enumerate(sigma.tolist()):
        v += float(a[i, j])
    return v


def check_anytime(rep, full, a=None, value_fn=None):
    sig = rep.assignment.sigma
    n = len(sig)
    assert rep.terminated_by == "deadline"
    assert sorted(sig.tolist()) == list(range(n))
    assert np.array_equal(rep.assignment.tau[sig], np.arange(n))
    want = ordered_objective(a, sig) if a is not None else value_fn(sig)
    assert rep.assignment.value == want
    tr = rep.objective_trace
    assert tr[0][0] == 0
    assert all(tr[k][0] < tr[k + 1][0] for k in range(len(tr) - 1))
    assert all(tr[k][1] <= tr[k + 1][1] for k in range(len(tr) - 1))
    # cut inside the first pass: only the device-side check does that
    assert rep.outer_iterations == 1
    assert rep.gpu["inner_iterations"] < full.gpu["inner_iterations"]
    assert rep.switches_applied < full.switches_applied


@pytest.mark.parametrize("graph", [True, False])
def test_deadline_mid_pass_c3(gpu_ctx, graph):
    """C3 (n = 10k P2P): 0.5 ms into a ~3 ms solve."""
    import paper_1106_5694_b200 as g
    gpu_ctx.generate("p2p", 10000, 0)
    a = gpu_ctx.read_rows(np.arange(10000))
    full = gpu_ctx.solve(g.ParallelConfig(seed=0, use_graph=graph))
    assert full.terminated_by == "converged"
    rep = gpu_ctx.solve(g.ParallelConfig(seed=0, use_graph=graph, deadline=500_000))
    check_anytime(rep, full, a)
    assert rep.switches_applied > 0


@pytest.mark.parametrize("graph", [True, False])
def test_deadline_mid_pass_c4(gpu_ctx, graph):
    """C4 (n = 30k fp32, generated on the device): 5 ms into the solve."""
    import paper_1106_5694_b200 as g
    n = 30000
    gpu_ctx.generate("f32", n, 0)
    full = gpu_ctx.solve(g.ParallelConfig(seed=0, use_graph=graph))
    rep = gpu_ctx.solve(g.ParallelConfig(seed=0, use_graph=graph, deadline=5_000_000))

    def value(sig):  # the ordered objective from the device copy, row by row
        v = 0.0
        for j0 in range(0, n, 2048):
            js = np.arange(j0, min(n, j0 + 2048))
            rows = gpu_ctx.read_rows(sig[js])
            for k, j in enumerate(js.tolist()):
                v += float(rows[k, j])
        return v

    check_anytime(rep, full, value_fn=value)
    assert rep.switches_applied > 0


def test_deadline_negative_budget_expires_at_once(gpu_ctx):
    """Deadline::starting with a negative budget is already expired: the
    initial assignment comes back (the C-ABI's -1 sentinel)."""
    import paper_1106_5694_b200 as g
    gpu_ctx.generate("int", 300, 2)
    rep = gpu_ctx.solve(g.ParallelConfig(seed=5, deadline=-7))
    assert rep.terminated_by == "deadline"
    assert rep.switches_applied == 0
    assert rep.objective_trace == [(0, rep.assignment.value)]


def _ranks(a, cfg, world, peer):
    import paper_1106_5694_b200 as g
    from paper_1106_5694_b200.dist import ThreadExchange, ThreadPeerExchange
    ex = (ThreadPeerExchange if peer else ThreadExchange).group(world)
    ctxs = [g.Context(0) for _ in range(world)]
    for c in ctxs:
        c.set_matrix(a)
    out, errs = [None] * world, []

    def run(r, cfgs):
        try:
            out[r] = [ctxs[r].solve(c, dist=ex[r]) for c in cfgs]
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
            ex[r].shared["barrier"].abort()

    th = [threading.Thread(target=run, args=(r, cfg)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(600)
    assert not any(t.is_alive() for t in th), "a rank hung"
    if peer:
        for e in ex:
            e.free()
    for c in ctxs:
        c.close()
    if errs:
        raise errs[0]
    return out


@pytest.mark.parametrize("peer,graph", [(True, True), (True, False), (False, False)])
def test_deadline_multi_rank_agrees(oracle, gpu_ctx, peer, graph):
    """Ranks stop at the same batch (identical sigma, value, trace) and the
    next solve on the same transport runs in step (epoch resynchronised) and
    equals the single-GPU result."""
    import paper_1106_5694_b200 as g
    a = oracle.generate("p2p", 6000, 3)
    gpu_ctx.set_matrix(a)
    full = gpu_ctx.solve(g.ParallelConfig(seed=1, use_graph=graph))
    cut = g.ParallelConfig(seed=1, use_graph=graph, deadline=1_000_000)
    again = g.ParallelConfig(seed=1, use_graph=graph)
    out = _ranks(a, [cut, again], 2, peer)
    r0, r1 = out[0][0], out[1][0]
    assert np.array_equal(r0.assignment.sigma, r1.assignment.sigma)
    assert r0.assignment.value == r1.assignment.value
    assert r0.objective_trace == r1.objective_trace
    assert r0.terminated_by == r1.terminated_by == "deadline"
    assert sorted(r0.assignment.sigma.tolist()) == list(range(6000))
    assert r0.assignment.value == ordered_objective(a, r0.assignment.sigma)
    assert r0.switches_applied < full.switches_applied
    for r in range(2):
        rep = out[r][1]
        assert rep.terminated_by == "converged"
        assert np.array_equal(rep.assignment.sigma, full.assignment.sigma)
        assert rep.assignment.value == full.assignment.value
