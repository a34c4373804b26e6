"""GPU suite against the golden fixtures the reference itself produced
(tests/golden/make_golden.py): every BASELINE config -- C1 int 1k, C2 int 5k,
C3 P2P 10k, fp32 10k, int 10k, C4 fp32 30k -- generated on the device with the
same splitmix64 recipes and solved through the C-ABI; sigma, tau, the value
bits, outer iterations, switches and the objective trace must be identical."""
import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "golden.json")))
ARR = np.load(os.path.join(HERE, "golden", "small_cases.npz"))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def trace_sha(trace):
    sw = np.array([t[0] for t in trace], np.int64)
    va = np.array([t[1] for t in trace], np.float64)
    return hashlib.sha256(sw.tobytes() + va.tobytes()).hexdigest()


def cfg(rec, **kw):
    import paper_1106_5694_b200 as g
    return g.ParallelConfig(seed=rec["seed"], improvement_epsilon=rec["eps"],
                            reeval="touched_only" if rec["policy"] else "touched_and_conflicted", **kw)


def check(rep, rec):
    assert sha(rep.assignment.sigma) == rec["sigma_sha"]
    assert sha(rep.assignment.tau) == rec["tau_sha"]
    assert float(rep.assignment.value).hex() == rec["value_hex"]
    assert rep.outer_iterations == rec["outer"]
    assert rep.switches_applied == rec["switches"]
    assert rep.terminated_by == rec["terminated_by"]
    assert len(rep.objective_trace) == rec["trace_len"]
    assert trace_sha(rep.objective_trace) == rec["trace_sha"]
    # the delta log was put in batch order on the device (log_order.cu)
    assert getattr(rep, "gpu", {}).get("host_log_orders", 0) == 0


@pytest.mark.parametrize("name", sorted(GOLD["solves"]))
def test_config_solves_bit_exact_vs_reference(gpu_ctx, name):
    rec = GOLD["solves"][name]
    gpu_ctx.generate(rec["kind"], rec["n"], rec["instance_seed"], rec["param"])
    check(gpu_ctx.solve(cfg(rec)), rec)


@pytest.mark.parametrize("name", sorted(GOLD["small"]))
@pytest.mark.parametrize("graph", [True, False])
def test_small_solves_bit_exact_vs_reference(oracle, gpu_ctx, name, graph):
    rec = GOLD["small"][name]
    if rec["kind"] == "explicit2":
        a = np.array([[0.0, 10.0], [10.0, 0.0]])
    else:
        a = oracle.generate(rec["kind"], rec["n"], rec["instance_seed"], rec["param"])
    gpu_ctx.set_matrix(a)
    rep = gpu_ctx.solve(cfg(rec, use_graph=graph))
    check(rep, rec)
    assert np.array_equal(rep.assignment.sigma, ARR[name + "__sigma"])


@pytest.mark.parametrize("key", sorted(GOLD["steps"]))
def test_step_apis_vs_reference(oracle, gpu_ctx, key):
    import paper_1106_5694_b200 as g
    rec = GOLD["steps"][key]
    n = rec["n"]
    a = oracle.generate(rec["kind"], n, rec["seed"])
    sigma = oracle.random_perm(n, rec["sigma_seed"])
    gpu_ctx.set_matrix(a)
    t = gpu_ctx.evaluate_all(sigma)
    for nm, v in (("ad", t.agent_delta), ("ap", t.agent_partner), ("jd", t.job_delta), ("jp", t.job_partner)):
        assert np.array_equal(np.asarray(v).view(np.uint8), ARR[f"{key}__{nm}"].view(np.uint8)), nm
    sets = gpu_ctx.check_conflicts(t, sigma)
    assert np.array_equal(sets.agent_accepted, ARR[f"{key}__acc_a"])
    assert np.array_equal(sets.job_accepted, ARR[f"{key}__acc_j"])
    assert sets.reserved == np.flatnonzero(ARR[f"{key}__reserved"]).tolist()
    assert sets.conflicted == np.flatnonzero(ARR[f"{key}__conflicted"]).tolist()
    assert sets.conflicted_jobs == ARR[f"{key}__cjobs"].tolist()
    gpu_ctx.set_matrix(a)  # check_conflicts may reuse the vectors
    tau = np.empty(n, np.int32)
    tau[sigma] = np.arange(n)
    value = float(np.cumsum(a[sigma, np.arange(n)])[-1])
    out, applied = gpu_ctx.apply_parallel_switches(g.Assignment(sigma, tau, value), t, sets)
    assert np.array_equal(out.sigma, ARR[f"{key}__sigma_after"])
    assert float(out.value).hex() == rec["value_after_hex"]
    assert [[x.agent, x.new_job, x.old_job, x.displaced] for x in applied] == ARR[f"{key}__applied"].tolist()
    assert [x.delta for x in applied] == ARR[f"{key}__applied_delta"].tolist()


@pytest.mark.parametrize("name", ["c1_int1000", "c2_int5000", "c3_p2p10000", "int10000", "f32_10000",
                                  "c2_int5000_touched_only", "geom2048"])
@pytest.mark.parametrize("graph", [True, False])
def test_config_solves_without_trace(gpu_ctx, name, graph):
    """The bench path (no trace buffers): integer storage replays the delta
    log as exact partial sums; results must still equal the reference's."""
    rec = GOLD["solves"][name]
    gpu_ctx.generate(rec["kind"], rec["n"], rec["instance_seed"], rec["param"])
    rep = gpu_ctx.solve(cfg(rec, use_graph=graph), trace=False)
    assert sha(rep.assignment.sigma) == rec["sigma_sha"]
    assert sha(rep.assignment.tau) == rec["tau_sha"]
    assert float(rep.assignment.value).hex() == rec["value_hex"]
    assert rep.outer_iterations == rec["outer"]
    assert rep.switches_applied == rec["switches"]
    assert rep.gpu["trace_len"] == rec["trace_len"]


ORDER_CASE = r'''
import sys, json, hashlib; sys.path.insert(0, %r)
import paper_1106_5694_b200 as g
ctx = g.Context(0)
out = {}
for kind, n, param in (("p2p", 3000, None), ("f32", 2500, None), ("geom", 2000, 100.0)):
    ctx.generate(kind, n, 1, param)
    for graph in (True, False):
        r = ctx.solve(g.ParallelConfig(seed=3, use_graph=graph))
        out["%%s-%%d-%%d" %% (kind, n, graph)] = [float(r.assignment.value).hex(), r.switches_applied,
            hashlib.sha256(repr(list(r.objective_trace)).encode()).hexdigest(), r.gpu["host_log_orders"]]
print(json.dumps(out))
'''


def test_device_log_order_equals_host_order():
    """The device-ordered delta log (log_order.cu) replays to the same trace
    and objective bits as the host's own ordering of the raw log
    (LSAPGPU_HOST_LOG_ORDER=1), for integer, fp32 and fp64 storage, graph
    and host-stepped passes."""
    import json, os, subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

    def run(env):
        r = subprocess.run([sys.executable, "-c", ORDER_CASE % root], env=dict(os.environ, **env),
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        return json.loads(r.stdout.strip().splitlines()[-1])

    dev, host = run({}), run({"LSAPGPU_HOST_LOG_ORDER": "1"})
    assert all(v[3] == 0 for v in dev.values()), dev
    assert all(v[3] > 0 for v in host.values()), host
    assert {k: v[:3] for k, v in dev.items()} == {k: v[:3] for k, v in host.items()}


DRAIN_CASE = r'''
import sys, json, hashlib; sys.path.insert(0, %r)
import paper_1106_5694_b200 as g
ctx = g.Context(0)
out = {}
for kind, n in (("p2p", 2000), ("f32", 1500)):
    ctx.generate(kind, n, 2)
    for graph in (True, False):
        for trace in (True, False):
            r = ctx.solve(g.ParallelConfig(seed=5, use_graph=graph), trace=trace)
            out["%%s-%%d-%%d" %% (kind, graph, trace)] = [float(r.assignment.value).hex(), r.switches_applied,
                hashlib.sha256(r.assignment.sigma.tobytes()).hexdigest(), r.outer_iterations,
                hashlib.sha256(repr(list(r.objective_trace)).encode()).hexdigest()]
print(json.dumps(out))
'''


def test_delta_log_drain_mid_pass():
    """A pass whose exchanges overflow the delta log drains it to the host and
    continues the inner loop (parallel.cpp has no such limit; the replay must
    not notice): with the log capped at ~2n entries (LSAPGPU_LOG_CAP) every
    solve -- graph / host-stepped, trace on / off, integer and fp32 storage --
    equals the uncapped one bit for bit, trace included."""
    import json, os, subprocess, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

    def run(env):
        r = subprocess.run([sys.executable, "-c", DRAIN_CASE % root], env=dict(os.environ, **env),
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        return json.loads(r.stdout.strip().splitlines()[-1])

    base, capped = run({}), run({"LSAPGPU_LOG_CAP": "1"})
    assert base == capped
