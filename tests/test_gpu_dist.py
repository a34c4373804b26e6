"""GPU: the multi-rank solve path on one device.  Each rank is
a thread with its own context; the allgather is device-to-device copies, so the
exact multi-GPU code path (item ownership by agent index, record pack / merge,
replicated commit) runs, and every rank must return the single-GPU result bit
for bit (which equals the reference's, see test_gpu_golden)."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def solve_ranks(a, cfg, world, peer=False):
    import paper_1106_5694_b200 as g
    from paper_1106_5694_b200.dist import ThreadExchange, ThreadPeerExchange
    ex = (ThreadPeerExchange if peer else ThreadExchange).group(world)
    out, errs = [None] * world, []

    def run(r):
        try:
            ctx = g.Context(0)
            ctx.set_matrix(a)
            out[r] = ctx.solve(cfg, dist=ex[r])
            ctx.close()
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
            ex[r].shared["barrier"].abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(600)
    if peer:
        for e in ex:
            e.free()
    if errs:
        raise errs[0]
    return out, ex


@pytest.mark.parametrize("kind,n,world,policy", [
    ("int", 1000, 2, "touched_and_conflicted"), ("geom", 500, 3, "touched_and_conflicted"),
    ("geom", 500, 2, "touched_only"), ("f32", 2000, 4, "touched_and_conflicted"), ("p2p", 1500, 8, "touched_and_conflicted"),
    ("int", 7, 4, "touched_and_conflicted")])
def test_multi_rank_equals_single_gpu(oracle, gpu_ctx, kind, n, world, policy):
    import paper_1106_5694_b200 as g
    a = oracle.generate(kind, n, 5)
    cfg = g.ParallelConfig(seed=3, reeval=policy)
    gpu_ctx.set_matrix(a)
    ref = gpu_ctx.solve(cfg)
    reps, ex = solve_ranks(a, cfg, world)
    assert all(e.calls > 0 for e in ex)
    for rep in reps:
        assert np.array_equal(rep.assignment.sigma, ref.assignment.sigma)
        assert rep.assignment.value == ref.assignment.value
        assert rep.objective_trace == ref.objective_trace
        assert rep.outer_iterations == ref.outer_iterations
        assert rep.gpu["inner_iterations"] == ref.gpu["inner_iterations"]


def test_torch_distributed_two_ranks(oracle, gpu_ctx, tmp_path):
    """The torch.distributed exchange (TorchDistExchange) across two real
    processes: gloo ranks sharing GPU 0, so the multi-process path bench.py
    uses at N > 1 (NCCL on a multi-GPU node) runs here end to end and must
    match the single-GPU solve bit for bit."""
    import os
    import subprocess
    import sys

    import paper_1106_5694_b200 as g
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    a = oracle.generate("int", 1500, 9)
    np.save(tmp_path / "a.npy", a)
    script = tmp_path / "rank.py"
    script.write_text(
        "import os, sys, numpy as np, torch, torch.distributed as dist\n"
        f"sys.path.insert(0, {root!r})\n"
        "import paper_1106_5694_b200 as g\n"
        "from paper_1106_5694_b200.dist import TorchDistExchange\n"
        "dist.init_process_group('gloo')\n"
        "torch.cuda.set_device(0)\n"
        f"a = np.load({str(tmp_path / 'a.npy')!r})\n"
        "ctx = g.Context(0); ctx.set_matrix(a)\n"
        "ex = TorchDistExchange()\n"
        "rep = ctx.solve(g.ParallelConfig(seed=4), dist=ex)\n"
        f"np.save(os.path.join({str(tmp_path)!r}, 'sigma%d.npy' % dist.get_rank()), rep.assignment.sigma)\n"
        "print('calls', ex.calls, 'value', rep.assignment.value)\n"
        "dist.destroy_process_group()\n")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29533", str(script)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    gpu_ctx.set_matrix(a)
    ref = gpu_ctx.solve(g.ParallelConfig(seed=4))
    for rank in range(2):
        sig = np.load(tmp_path / f"sigma{rank}.npy")
        assert np.array_equal(sig, ref.assignment.sigma)


@pytest.mark.parametrize("world", [2, 4])
def test_multi_rank_greedy_start(oracle, gpu_ctx, world):
    """Every rank computes the same (deterministic) greedy start on its replica."""
    import paper_1106_5694_b200 as g
    a = oracle.generate("p2p", 1200, 7)
    cfg = g.ParallelConfig(init="greedy")
    gpu_ctx.set_matrix(a)
    ref = gpu_ctx.solve(cfg)
    reps, _ = solve_ranks(a, cfg, world)
    for rep in reps:
        assert np.array_equal(rep.assignment.sigma, ref.assignment.sigma)
        assert rep.assignment.value == ref.assignment.value
        assert rep.objective_trace == ref.objective_trace


@pytest.mark.parametrize("kind,n,world,policy,graph", [
    ("int", 1000, 2, "touched_and_conflicted", True), ("geom", 500, 3, "touched_only", True),
    ("f32", 2000, 4, "touched_and_conflicted", True), ("int", 7, 4, "touched_and_conflicted", True),
    ("int", 1000, 2, "touched_and_conflicted", False), ("p2p", 1500, 8, "touched_and_conflicted", False)])
def test_peer_transport_equals_single_gpu(oracle, gpu_ctx, kind, n, world, policy, graph):
    """The peer-memory transport (records pushed into every replica by the
    pack kernel, epoch flags, no allgather call) with ranks as threads on one
    device: bit-identical to the single-GPU solve, repeated solves included
    (the epochs continue across solves).  Graph mode (the whole batch loop in
    one graph launch per rank) is emulated with at most 4 ranks sharing the
    device: more graphs spinning on peer flags on ONE GPU can starve each
    other's device-side launches (with one process per GPU nothing is shared);
    8 ranks run host-stepped."""
    import paper_1106_5694_b200 as g
    from paper_1106_5694_b200.dist import ThreadPeerExchange
    a = oracle.generate(kind, n, 5)
    cfg = g.ParallelConfig(seed=3, reeval=policy, use_graph=graph)
    gpu_ctx.set_matrix(a)
    ref = gpu_ctx.solve(cfg)
    ex = ThreadPeerExchange.group(world)
    out, errs = [None] * world, []

    def run(r):
        try:
            ctx = g.Context(0)
            ctx.set_matrix(a)
            out[r] = [ctx.solve(cfg, dist=ex[r]) for _ in range(2)]
            ctx.close()
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
            ex[r].shared["barrier"].abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(600)
    for e in ex:
        e.free()
    if errs:
        raise errs[0]
    for reps in out:
        for rep in reps:
            assert np.array_equal(rep.assignment.sigma, ref.assignment.sigma)
            assert rep.assignment.value == ref.assignment.value
            assert rep.objective_trace == ref.objective_trace
            assert rep.gpu["inner_iterations"] == ref.gpu["inner_iterations"]


def test_peer_transport_two_processes_ipc(oracle, gpu_ctx, tmp_path):
    """TorchPeerExchange across two real processes (CUDA IPC mappings of each
    other's buffers, here on one device; NVLink peers on a multi-GPU node)."""
    import os
    import subprocess
    import sys

    import paper_1106_5694_b200 as g
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    a = oracle.generate("p2p", 1200, 11)
    np.save(tmp_path / "a.npy", a)
    script = tmp_path / "rank.py"
    script.write_text(
        "import os, sys, numpy as np, torch, torch.distributed as dist\n"
        f"sys.path.insert(0, {root!r})\n"
        "import paper_1106_5694_b200 as g\n"
        "from paper_1106_5694_b200.dist import TorchPeerExchange\n"
        "dist.init_process_group('gloo')\n"
        "torch.cuda.set_device(0)\n"
        f"a = np.load({str(tmp_path / 'a.npy')!r})\n"
        "ctx = g.Context(0); ctx.set_matrix(a)\n"
        "ex = TorchPeerExchange()\n"
        "rep = ctx.solve(g.ParallelConfig(seed=6), dist=ex)\n"
        "rep = ctx.solve(g.ParallelConfig(seed=6), dist=ex)\n"
        f"np.save(os.path.join({str(tmp_path)!r}, 'sigma%d.npy' % dist.get_rank()), rep.assignment.sigma)\n"
        "dist.barrier(); ex.close(); ctx.close()\n"
        "dist.destroy_process_group()\n")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29534", str(script)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    gpu_ctx.set_matrix(a)
    ref = gpu_ctx.solve(g.ParallelConfig(seed=6))
    for rank in range(2):
        assert np.array_equal(np.load(tmp_path / f"sigma{rank}.npy"), ref.assignment.sigma)


@pytest.mark.parametrize("exchange", ["nccl", "p2p"])
def test_bench_two_ranks_sharded_block(tmp_path, exchange):
    """bench.py at N = 2 (torchrun, gloo, both ranks on GPU 0): one JSON line
    with the sharded C4 block of the metric's multi-GPU config -- the
    sharded n = 30k solve must reproduce the reference's golden sigma
    (tests/golden c4_f32_30000) and report its per-N sweep time and the
    transport used."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    port = "29541" if exchange == "nccl" else "29542"
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", port, os.path.join(root, "bench.py"),
                        "--gpus", "2", "--backend", "gloo", "--exchange", exchange, "--steps", "2", "--warmup", "3",
                        "--workload", "c1", "--blocks", "c4"],
                       capture_output=True, text=True, timeout=1200, cwd=str(tmp_path))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2 and out["scaling"] == "strong"
    blk = out["sharded"]["c4"]
    assert "error" not in blk, blk
    assert blk["n_gpus"] == 2 and blk["items_per_rank"] == 15000
    assert blk["sigma_sha_matches_golden"] is True
    assert blk["full_sweep_ms"] > 0 and blk["scan_kernel"] == "filter"
    assert ("peer-memory" in blk["transport"]) == (exchange == "p2p")


def test_sharded_large_filter_equals_single_gpu(tmp_path):
    """The sharded solve at a C5-like size on the filter scan (n = 60000
    fp32, int8 copies, each rank scanning its share of the items): both
    ranks return the single-GPU sigma bit for bit (peer transport, ranks as
    threads on GPU 0 -- two 36 GB replicas)."""
    import hashlib
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys, json, hashlib, threading; sys.path.insert(0, %r)\n"
        "import paper_1106_5694_b200 as g\n"
        "from paper_1106_5694_b200.dist import ThreadPeerExchange\n"
        "n = 60000\n"
        "h = lambda s: hashlib.sha256(s.tobytes()).hexdigest()\n"
        "ctx = g.Context(0); ctx.generate('f32', n, 0)\n"
        "ref = ctx.solve(g.ParallelConfig(seed=0)); plan = ctx.scan_plan(); ctx.close()\n"
        "ex = ThreadPeerExchange.group(2); out = [None, None]\n"
        "def run(r):\n"
        "    c = g.Context(0); c.generate('f32', n, 0)\n"
        "    out[r] = c.solve(g.ParallelConfig(seed=0), dist=ex[r]); c.close()\n"
        "th = [threading.Thread(target=run, args=(r,)) for r in range(2)]\n"
        "[t.start() for t in th]; [t.join() for t in th]\n"
        "[e.free() for e in ex]\n"
        "print(json.dumps({'plan': plan, 'ref': h(ref.assignment.sigma), 'value': ref.assignment.value,\n"
        "                  'ranks': [h(o.assignment.sigma) for o in out], 'values': [o.assignment.value for o in out]}))\n"
        % root)
    env = dict(os.environ, LSAPGPU_FILTER_BITS="8")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    out = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert out["plan"]["kernel"] == "filter" and out["plan"]["filter"] == 8
    assert out["ranks"] == [out["ref"], out["ref"]]
    assert out["values"] == [out["value"], out["value"]]


@pytest.mark.parametrize("kind,n,world,peer,graph", [
    ("p2p", 1500, 2, True, True),      # resident scan
    ("int", 997, 3, False, False),     # ragged blocks, allgather transport, host-stepped
    ("f32", 12000, 2, True, True),     # filter scan on the row block's Q rows
    ("geom", 700, 4, True, False),     # fp64
])
def test_row_block_placement_equals_single_gpu(oracle, gpu_ctx, kind, n, world, peer, graph):
    """Row-block placement (lsapgpu_set_placement, SURVEY §8(e) placement
    (i)): each rank holds only its agents' rows of A (and Q) plus all of AT;
    every rank returns the single-GPU result bit for bit, and single-GPU entry
    points refuse such a context."""
    import paper_1106_5694_b200 as g
    from paper_1106_5694_b200.dist import ThreadExchange, ThreadPeerExchange
    a = oracle.generate(kind, n, 8)
    cfg = g.ParallelConfig(seed=2, use_graph=graph)
    gpu_ctx.set_matrix(a)
    ref = gpu_ctx.solve(cfg)
    ex = (ThreadPeerExchange if peer else ThreadExchange).group(world)
    out, errs = [None] * world, []

    def run(r):
        try:
            ctx = g.Context(0)
            ctx.set_placement(r, world)
            ctx.set_matrix(a)
            out[r] = [ctx.solve(cfg, dist=ex[r]) for _ in range(2)]
            with pytest.raises(g.Error, match="row block"):
                ctx.solve(cfg)
            ctx.close()
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
            ex[r].shared["barrier"].abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(600)
    if peer:
        for e in ex:
            e.free()
    if errs:
        raise errs[0]
    for reps in out:
        for rep in reps:
            assert np.array_equal(rep.assignment.sigma, ref.assignment.sigma)
            assert rep.assignment.value == ref.assignment.value
            assert rep.objective_trace == ref.objective_trace
