"""CPU, world_size 2 over gloo: the multi-GPU decomposition of DESIGN.md §7
(the protocol csrc/dist.cu implements) restated over the oracle's step
functions.  Each rank owns the work items of agents i with i % world == rank,
evaluates only their records, packs them in the 32-byte record layout of
dist.cu, allgathers over torch.distributed (gloo), merges every rank's records
and runs the conflict check / apply replicated.  Both ranks must reach the
single-process reference result bit for bit, for both re-evaluation policies.
"""
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

REC = np.dtype([("agent", "<i4"), ("job", "<i4"), ("ap", "<i4"), ("jp", "<i4"), ("ad", "<f8"), ("jd", "<f8")])
assert REC.itemsize == 32


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def distributed_dgs(oracle, a, seed, policy, rank, world, allgather):
    """Restatement of parallel.cpp:231-352 where every evaluation is partitioned
    by agent owner and exchanged (test infrastructure)."""
    n = a.shape[0]
    sigma = oracle.random_perm(n, seed)
    tau = np.empty(n, np.int32)
    tau[sigma] = np.arange(n)
    value = float(np.cumsum(a[sigma, np.arange(n)])[-1])
    ad, jd = np.zeros(n), np.zeros(n)
    ap, jp = np.full(n, -1, np.int32), np.full(n, -1, np.int32)
    trace = [(0, value)]
    switches = outer = 0

    def scan(items):  # items: {agent: (agent_flag, job_flag)}
        fad, fap, fjd, fjp = oracle.evaluate_all(a, sigma)  # records on the frozen state
        mine = [i for i in sorted(items) if i % world == rank]
        buf = np.zeros(len(mine), REC)
        for k, i in enumerate(mine):
            af, jf = items[i]
            j = tau[i]
            buf[k] = (i if af else -2 - i, j if jf else -1, fap[i], fjp[j], fad[i], fjd[j])
        for rec in allgather(buf):  # every rank's records, merged identically
            for r in rec:
                if r["agent"] >= 0:
                    ad[r["agent"]], ap[r["agent"]] = r["ad"], r["ap"]
                if r["job"] >= 0:
                    jd[r["job"]], jp[r["job"]] = r["jd"], r["jp"]

    while True:
        outer += 1
        f_start = value
        scan({i: (True, True) for i in range(n)})
        while (ad > 0).any() or (jd > 0).any():
            cc = oracle.check_conflicts(ad, ap, jd, jp, sigma)
            batch = []
            for side, acc, dd, pp in ((0, cc["agent_accepted"], ad, ap), (1, cc["job_accepted"], jd, jp)):
                for k in np.flatnonzero(acc):
                    partner = int(pp[k])
                    dd[k], pp[k] = 0.0, -1
                    if side == 0:
                        i, jn = int(k), partner
                        jo, d = int(tau[i]), int(sigma[jn])
                        act = (a[i, jn] - a[i, jo]) + (a[d, jo] - a[d, jn])
                    else:
                        i, jn = partner, int(k)
                        h, jo = int(sigma[jn]), int(tau[partner])
                        d = h
                        act = (a[i, jn] - a[h, jn]) + (a[h, jo] - a[i, jo])
                    if act > 0.0:
                        batch.append((i, jn, jo, d, act))
            touched = set()
            for i, jn, jo, d, act in batch:
                sigma[jn], sigma[jo], tau[i], tau[d] = i, d, jn, jo
                value += act
                switches += 1
                trace.append((switches, value))
                touched |= {i, d}
            items = {i: (True, True) for i in touched}
            if policy == 0:
                cj = set(cc["conflicted_jobs"].tolist())
                for i in np.flatnonzero(cc["conflicted"]):
                    if int(i) not in touched:
                        items[int(i)] = (True, int(tau[i]) in cj)
            scan(items)
        if value == f_start:
            break
    return sigma, value, trace, outer


def _worker(rank, world, port, q):
    import torch
    from oracle.oracle import Oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    oracle = Oracle()

    def allgather(buf):
        raw = torch.from_numpy(buf.view(np.uint8).copy())
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([raw.numel()], dtype=torch.int64))
        cap = int(max(s.item() for s in sizes))
        pad = torch.zeros(cap, dtype=torch.uint8)
        pad[:raw.numel()] = raw
        outs = [torch.zeros(cap, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(outs, pad)
        return [o[:int(s.item())].numpy().view(REC) for o, s in zip(outs, sizes)]

    results = []
    for kind, n, seed, policy in (("int", 60, 3, 0), ("geom", 48, 4, 0), ("geom", 48, 4, 1), ("f32", 40, 9, 0)):
        a = oracle.generate(kind, n, 11)
        s, v, tr, outer = distributed_dgs(oracle, a, seed, policy, rank, world, allgather)
        results.append((s.tolist(), v, tr, outer))
    q.put((rank, results))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_protocol_matches_reference(oracle):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    cases = (("int", 60, 3, 0), ("geom", 48, 4, 0), ("geom", 48, 4, 1), ("f32", 40, 9, 0))
    for k, (kind, n, seed, policy) in enumerate(cases):
        ref = oracle.dgs_parallel(oracle.generate(kind, n, 11), seed=seed, policy=policy)
        for r in range(world):
            s, v, tr, outer = got[r][k]
            assert s == ref.sigma.tolist(), (kind, policy, r)
            assert v == ref.trace[-1][1]  # the running value the reference accumulates
            assert tr == ref.trace
            assert outer == ref.outer_iterations
