#!/usr/bin/env python3
"""Benchmark: LSAP time-to-solution (ms) of the B200 DGS solver.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c3|c1|c2|c4|c5]

Workload (BASELINE.json metric "LSAP time-to-solution ms at n=10k (1 B200)"):
C3, the n=10000 P2P-streaming-shaped integer matrix, instance
seed 0, solver seed 0, default ParallelConfig.

One step = one full ``dgs_parallel`` solve of that instance:
  value : input fp64 matrix already resident in HBM -> validate/classify,
          narrow + transpose (A, AT), initial assignment, every outer/inner
          iteration, sigma/tau back on the host (CUDA events on the solver's
          stream, synchronize on both sides).
  e2e   : the same call through the public C-ABI with the fp64 matrix in
          pinned HOST memory: H2D of the 8*n^2-byte input + solve + D2H of the
          result, all inside the timed region.
Inputs (800 MB fp64 + 200 MB int16 A/AT at C3) exceed the 126 MB L2, so no
extra flush is needed between steps.

--impl reference times the reference's own CPU implementation
(oracle/_ref/liblsap_ref.so = the unmodified reference sources compiled by
oracle/Makefile; falls back to the C restatement oracle/liboracle.so) on the
same instance with all host threads.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (kind, n, instance seed, param, description)
    "c1": ("int", 1000, 0, 1000.0, "n=1000 uniform integer benefits in [0,1000), seed 0"),
    "c2": ("int", 5000, 0, 1000.0, "n=5000 uniform integer benefits in [0,1000), seed 0"),
    "c3": ("p2p", 10000, 0, None, "n=10000 P2P-streaming-shaped benefit matrix, seed 0"),
    "c4": ("f32", 30000, 0, None, "n=30000 fp32 uniform random benefits in [0,1], seed 0"),
    "c5": ("f32", 100000, 0, None, "n=100000 fp32 uniform random benefits in [0,1], seed 0"),
}
METRIC = "LSAP time-to-solution ms at n=10k (1 B200) + sweep HBM GB/s; 2/4/8-GPU at n=100k"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            t0 = time.time()  # the first sample takes a while: start timing only once it arrived
            while not self.lines and time.time() - t0 < 3.0 and self.proc.poll() is None:
                time.sleep(0.01)
            self.pre = list(self.lines)  # warm-up samples: used only if the region saw none
            self.lines.clear()
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sms, maxes, reasons = [], [], set()
        if not self.lines:
            self.lines = getattr(self, "pre", [])
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sms.append(float(parts[1]))
                maxes.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sms:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sms), "sm_max_mhz": max(maxes), "reasons": sorted(reasons),
                "samples": len(sms)}


def measured_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json, burst copy)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def ncu_traffic(workload: str) -> dict | None:
    """DRAM bytes per launch of this workload's pair-scan kernel (one full
    sweep) from the committed ncu --set full summaries, keyed by workload,
    beside the algorithmic bytes of the same launch."""
    p = os.path.join(ROOT, "profiles", "ncu_pair_scan_summary.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    return d.get(workload)


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------
def run_reference(args, wl) -> None:
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle.oracle import Oracle, load_ref_or_none
    kind, n, iseed, param, desc = wl
    orc = Oracle()
    ref = load_ref_or_none()
    a = orc.generate(kind, n, iseed, param)
    cores = os.cpu_count() or 1
    times = []
    for k in range(args.warmup + args.steps):
        if ref is not None:
            r = ref.dgs_parallel(a, seed=0, workers=cores, trace=False)
        else:
            r = orc.dgs_parallel(a, seed=0, threads=cores, trace=False)
        if k >= args.warmup:
            times.append(r.elapsed_ms)
    kind_s = "reference" if ref is not None else "port"
    v = statistics.median(times)
    out = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "ms", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": v, "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": desc, "n": n, "solver_seed": 0, "reeval": "touched_and_conflicted",
                   "engine": "lsap::dgs_parallel (CPU, workers = all host threads)"},
        "cpu_baseline": {"value": v, "unit": "ms", "cores": cores, "kind": kind_s,
                         "sample": f"one full dgs_parallel solve of {desc} per step "
                                   f"(SolveReport.elapsed: validate + transpose + solve), median of {args.steps}"},
        "e2e": {"value": v, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "objective": r.value, "switches": r.switches_applied, "outer_iterations": r.outer_iterations,
    }
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def cpu_baseline(wl) -> dict:
    """The reference CPU path on this host, one bounded solve of the same workload."""
    from oracle.oracle import Oracle, load_ref_or_none
    kind, n, iseed, param, desc = wl
    orc = Oracle()
    ref = load_ref_or_none()
    a = orc.generate(kind, n, iseed, param)
    cores = os.cpu_count() or 1
    if ref is not None:
        r = ref.dgs_parallel(a, seed=0, workers=cores, trace=False)
        kind_s = "reference"
    else:
        r = orc.dgs_parallel(a, seed=0, threads=cores, trace=False)
        kind_s = "port"
    return {"value": r.elapsed_ms, "unit": "ms", "cores": cores, "kind": kind_s,
            "sample": f"one full dgs_parallel solve of {desc} (SolveReport.elapsed), same instance",
            "objective": r.value, "sigma_sha_matches_gpu": None, "_sigma": r.sigma}


def _allmax(x: float, world: int, backend: str, local: int) -> float:
    if world == 1:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}" if backend == "nccl" else "cpu")
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def _make_exchange(ctx, args):
    """The multi-rank record exchange: peer-memory push (NVLink P2P through
    CUDA IPC mappings) or, if that cannot be set up, a torch.distributed
    allgather (NCCL)."""
    from paper_1106_5694_b200.dist import TorchDistExchange, TorchPeerExchange
    exch, transport = None, None
    if args.exchange == "p2p":
        try:
            exch = TorchPeerExchange()
            exch.struct(ctx)
            transport = "peer-memory push (pack + allgather in one kernel, CUDA IPC over NVLink)"
        except Exception as e:  # noqa: BLE001
            exch = None
            transport = f"{args.backend} allgather (peer transport unavailable: {e})"
    if exch is None:
        exch = TorchDistExchange()
        transport = transport or f"{args.backend} allgather"
    return exch, transport


def _close_exchange(exch):
    for m in ("close", "free"):
        f = getattr(exch, m, None)
        if f is not None:
            try:
                f()
            except Exception:  # noqa: BLE001
                pass
            return


def golden_solves() -> dict:
    p = os.path.join(ROOT, "tests", "golden", "golden.json")
    if not os.path.exists(p):
        return {}
    with open(p) as f:
        return json.load(f).get("solves", {})


def sweep_block(g, args, wname: str, world: int, rank: int, local: int) -> dict:
    """The sharded solve of one BASELINE config at this N (C4: n = 30k, C5:
    n = 100k, both fp32 generated on the device): time to solution (max over
    ranks), the full-sweep time of the pair scan (each rank scans its share of
    the items; max over ranks) and its HBM rate, sigma against the golden
    fixture where one exists.  At N = 1 it is the plain single-GPU solve."""
    import hashlib

    import numpy as np
    import torch
    kind, n, iseed, param, desc = WORKLOADS[wname]
    ctx = g.Context(local)
    exch = transport = None
    try:
        if world > 1 and args.placement == "rows":
            ctx.set_placement(rank, world)  # this rank's row block of A + all of AT
        ctx.generate(kind, n, iseed, param)
        if world > 1:
            exch, transport = _make_exchange(ctx, args)
        cfg = g.ParallelConfig(seed=0)
        stream = torch.cuda.ExternalStream(ctx.stream)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        rep = ctx.solve(cfg, dist=exch)  # warm-up (graphs, plans)
        times = []
        for _ in range(2):
            if world > 1:
                torch.distributed.barrier()
            torch.cuda.synchronize()
            ev0.record(stream)
            rep = ctx.solve(cfg, dist=exch)
            ev1.record(stream)
            ev1.synchronize()
            times.append(ev0.elapsed_time(ev1))
        ms = _allmax(statistics.mean(times), world, args.backend, local)
        # instrumented host-stepped solve: CUDA events around every scan launch of this rank
        ctx.set_scan_timing(True)
        ctx.solve(g.ParallelConfig(seed=0, use_graph=False), dist=exch)
        ctx.set_scan_timing(False)
        tm = ctx.scan_timing()
        full_ms = _allmax(tm["full_ms"] / max(tm["full_launches"], 1), world, args.backend, local)
        plan = ctx.scan_plan()
        eb = ctx.storage_bytes
        qb = plan["filter"] // 8 if plan["filter"] else eb
        own = (n + world - 1) // world  # items of the most loaded rank (agent i -> rank i % N)
        alg = 2.0 * n * eb * n          # 2 n sizeof(elem) per item, all ranks
        hbm = 2.0 * n * qb * n          # bytes the kernel actually streams (quantized copies)
        pk = measured_peaks()["hbm_gbs"]
        sig_sha = hashlib.sha256(np.ascontiguousarray(rep.assignment.sigma).tobytes()).hexdigest()
        gold = golden_solves().get({"c4": "c4_f32_30000"}.get(wname, ""), None)
        return {
            "workload": desc, "n": n, "n_gpus": world, "ms": ms, "step_ms_all": times,
            "transport": transport if world > 1 else "none (one GPU)",
            "placement": ("row blocks of A + AT replicated" if args.placement == "rows" else "full A + AT replicas")
                         if world > 1 else "single",
            "full_sweep_ms": full_ms, "items_per_rank": own,
            "full_sweep_algorithmic_gbs": alg / (full_ms * 1e-3) / 1e9,
            "full_sweep_frac": alg / (full_ms * 1e-3) / 1e9 / pk,
            "full_sweep_hbm_gbs": hbm / (full_ms * 1e-3) / 1e9,
            "scan_kernel": plan["kernel"], "filter_bits": plan["filter"],
            "objective": rep.assignment.value, "switches": rep.switches_applied,
            "outer_iterations": rep.outer_iterations, "inner_iterations": rep.gpu["inner_iterations"],
            "filter_kept_per_item": rep.gpu["filter_kept"] / max(rep.gpu["pair_items"], 1),
            "sigma_sha": sig_sha,
            "sigma_sha_matches_golden": (sig_sha == gold["sigma_sha"]) if gold else None,
        }
    finally:
        if exch is not None:
            _close_exchange(exch)
        ctx.close()
        torch.cuda.synchronize()


def run_ours(args, wl) -> None:
    import numpy as np
    import torch

    rank, world, local = dist_env()
    if args.backend == "gloo":
        local = 0  # every rank on GPU 0 (tests of the multi-rank path on one device)
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if args.backend == "nccl":
            # communicator logging (stderr-free of our JSON): one INIT line per rank with nRanks
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:  # gloo: several ranks sharing one GPU (tests of the sharded path)
            dist.init_process_group("gloo")
    torch.cuda.set_device(local)
    import paper_1106_5694_b200 as g

    kind, n, iseed, param, desc = wl
    # N > 1: by default ONE instance is solved by all ranks (the sharded solve
    # of DESIGN.md §7: scan items owned by agent index, per-batch record
    # exchange, replicated commit); --replicas: every rank solves its own
    # instance (seed offset by rank)
    sharded = world > 1 and not args.replicas
    if world > 1 and not sharded:
        iseed = iseed + rank
    ctx = g.Context(local)
    if sharded and args.placement == "rows":
        ctx.set_placement(rank, world)
    cfg = g.ParallelConfig(seed=0)
    stream = torch.cuda.ExternalStream(ctx.stream)
    exch = None
    transport = None

    def solve():
        # trace on: the reference always builds the objective trace (parallel.cpp:15-20)
        return ctx.solve(cfg, dist=exch)

    # the input instance (fp64 host matrix, like lsap::Instance), built by the
    # package's on-device generator (same recipe and bits as the reference's)
    if n <= 30000:
        a_host = torch.from_numpy(g.generate_instance(kind, n, iseed, param, device=local)).pin_memory()
    else:
        ctx.generate(kind, n, iseed, param)  # too big for a host fp64 copy; build on device
        a_host = None
    a_dev = a_host.to(f"cuda:{local}") if a_host is not None else None
    torch.cuda.synchronize()
    if sharded:
        if a_dev is not None:
            ctx.set_matrix(a_dev)  # exchange buffers are sized for n
        exch, transport = _make_exchange(ctx, args)

    def step_device():
        ctx.set_matrix(a_dev)
        return solve()

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def timed(step, k, strm=None):
        strm = strm or stream
        times = []
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        rep = None
        for _ in range(k):
            barrier()
            ev0.record(strm)
            rep = step()
            ev1.record(strm)
            ev1.synchronize()
            times.append(ev0.elapsed_time(ev1))
        return times, rep

    step = step_device if a_dev is not None else solve
    for _ in range(args.warmup):
        step()
    c0 = ctx.counters()
    with ClockSampler(local) as clk:
        barrier()
        times, rep = timed(step, args.steps)
        barrier()
    c1 = ctx.counters()
    ms = _allmax(statistics.mean(times), world, args.backend, local)
    launches = (c1["kernel_launches"] - c0["kernel_launches"]) // max(args.steps, 1)

    # e2e through the public API, host fp64 input, copies inside the timed
    # region.  One GPU: the drop-in entry point lsap.dgs_parallel(Instance,
    # ParallelConfig) -- what a caller of the reference's API switches to --
    # with a plain (pageable) numpy Instance and the objective trace on.
    # N > 1: set_matrix(host) + the sharded solve on every rank.
    e2e = None
    if a_host is not None:
        a_pageable = a_host.numpy().copy()
        if world == 1:
            inst = g.Instance(n, a_pageable)
            dctx = g.context(local)  # the context lsap.dgs_parallel uses on this thread
            dstream = torch.cuda.ExternalStream(dctx.stream)
            dcfg = g.ParallelConfig(seed=0, device=local)

            def step_e2e():
                return g.dgs_parallel(inst, dcfg)

            entry = "lsap.dgs_parallel(Instance(pageable fp64 numpy), ParallelConfig(seed=0)), trace on"
        else:
            dctx, dstream = ctx, stream

            def step_e2e():
                ctx.set_matrix(a_pageable)
                return solve()

            entry = "Context.set_matrix(pageable fp64) + sharded Context.solve(dist=...)"
        for _ in range(max(1, args.warmup // 2)):
            step_e2e()
        e0 = dctx.counters()
        etimes, erep = timed(step_e2e, args.steps, dstream)
        e1 = dctx.counters()
        e2e_ms = _allmax(statistics.mean(etimes), world, args.backend, local)
        e2e = {"value": e2e_ms, "unit": "ms",
               "h2d_bytes_per_step": (e1["h2d_bytes"] - e0["h2d_bytes"]) // args.steps,
               "d2h_bytes_per_step": (e1["d2h_bytes"] - e0["d2h_bytes"]) // args.steps,
               "source": entry,
               "sigma_matches_value_run": bool(np.array_equal(erep.assignment.sigma, rep.assignment.sigma)),
               "step_ms_all": etimes}
        # the same matrix from a pinned host buffer through the C-ABI
        pin = a_host.numpy()

        def step_pinned():
            ctx.set_matrix(pin)
            return solve()

        step_pinned()
        ptimes, _ = timed(step_pinned, max(1, min(args.steps, 5)))
        e2e["pinned_ms"] = _allmax(statistics.mean(ptimes), world, args.backend, local)

    # roofline of the dominant kernel (pair scan): instrumented host-stepped solve,
    # every scan launch bracketed by CUDA events on the solver's stream
    ctx.set_scan_timing(True)
    trep = ctx.solve(g.ParallelConfig(seed=0, use_graph=False), dist=exch)
    ctx.set_scan_timing(False)
    tm = ctx.scan_timing()
    plan = ctx.scan_plan()
    eb = ctx.storage_bytes
    pk = measured_peaks()
    kname = {"resident": "pair_scan_res_kernel", "streaming": "pair_scan_kernel",
             "filter": "pair_scan_filter_kernel"}[plan["kernel"]]
    full_bytes = n * 2 * n * eb / (world if sharded else 1)
    scan_bytes = trep.gpu["bytes_scanned"] / (world if sharded else 1)
    achieved_all = scan_bytes / (tm["scan_ms"] * 1e-3) / 1e9 if tm["scan_ms"] > 0 else None
    achieved_full = (full_bytes * tm["full_launches"]) / (tm["full_ms"] * 1e-3) / 1e9 if tm["full_ms"] > 0 else None
    tr = ncu_traffic(args.workload)
    roofline = {
        "bound": "hbm", "achieved": achieved_all, "peak": pk["hbm_gbs"], "unit": "GB/s",
        "frac": achieved_all / pk["hbm_gbs"] if achieved_all else None,
        "traffic": tr.get("dram_bytes_per_launch") if tr else None,
        "traffic_algorithmic_bytes": tr.get("algorithmic_bytes_per_launch") if tr else None,
        "kernel": f"{kname} (all launches of one solve: full sweeps + re-evaluation lists)",
        "algorithmic_bytes_per_launch": scan_bytes / max(tm["scan_launches"], 1),
        "avg_launch_ms": tm["scan_ms"] / max(tm["scan_launches"], 1),
        "full_sweep": {"achieved": achieved_full, "frac": achieved_full / pk["hbm_gbs"] if achieved_full else None,
                       "bytes_per_launch": full_bytes, "avg_launch_ms": tm["full_ms"] / max(tm["full_launches"], 1)},
        "scan_share_of_solve": tm["scan_ms"] / trep.elapsed * 1e6 if trep.elapsed else None,
        "peak_source": pk["source"],
        "traffic_source": tr.get("source") if tr else None,
        "plan": plan,
    }
    if plan["filter"]:  # the filter kernel streams quantized copies: its actual rate beside the algorithmic one
        qbytes = full_bytes * (plan["filter"] // 8) / eb
        roofline["full_sweep"]["streamed_bytes_per_launch"] = qbytes
        roofline["full_sweep"]["streamed_gbs"] = (qbytes * tm["full_launches"]) / (tm["full_ms"] * 1e-3) / 1e9 \
            if tm["full_ms"] > 0 else None

    # extension (not the headline): the same step from the device greedy
    # initial assignment instead of the reference's initial_random; its result
    # differs from the reference's (DGS from another start), so it is reported
    # beside the reference-identical measurement
    greedy = None
    if world == 1:
        gcfg = g.ParallelConfig(seed=0, init="greedy")

        def step_greedy():
            if a_dev is not None:
                ctx.set_matrix(a_dev)
            return ctx.solve(gcfg)

        for _ in range(2):
            step_greedy()
        gtimes, grep = timed(step_greedy, args.steps)
        greedy = {"value": statistics.mean(gtimes), "unit": "ms", "objective": grep.assignment.value,
                  "objective_vs_reference_start": grep.assignment.value - rep.assignment.value,
                  "switches": grep.switches_applied, "inner_iterations": grep.gpu["inner_iterations"],
                  "solve_ms_internal": grep.elapsed / 1e6,
                  "note": "ParallelConfig(init='greedy'): device greedy initial assignment (north-star "
                          "item 2, not in the reference) then the same dgs_parallel loop"}

    # correctness of the measured run vs the oracle/reference (rank 0 only), and the CPU baseline
    cpu = None
    if rank == 0 and world == 1 and a_host is not None and not args.no_cpu:
        cpu = cpu_baseline(wl)
        sig = cpu.pop("_sigma")
        cpu["sigma_sha_matches_gpu"] = bool(np.array_equal(sig, rep.assignment.sigma))
        cpu["objective_matches_gpu"] = cpu.pop("objective") == rep.assignment.value

    clocks = clk.summary()
    if exch is not None:
        _close_exchange(exch)
        exch = None
    ctx.close()
    torch.cuda.synchronize()

    # the metric's multi-GPU configs (BASELINE configs[3] C4, configs[4] C5):
    # the sharded solve and sweep at this N, beside the C3 headline
    blocks = {}
    for wname in [w for w in args.blocks.split(",") if w]:
        try:
            blocks[wname] = sweep_block(g, args, wname, world, rank, local)
        except Exception as e:  # noqa: BLE001 -- reported, never silently dropped
            blocks[wname] = {"error": f"{type(e).__name__}: {e}"}
            if world > 1:
                raise

    out = {
        "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
        "scaling": "strong" if sharded else "weak",
        "vs_baseline": None, "dtype": {"int16": "i16->i32", "int32": "i32", "fp32": "f32->f64",
                                       "fp64": "f64"}[rep.gpu["storage"]],
        "data": "synthetic",
        "config": {"workload": desc, "n": n, "solver_seed": 0, "reeval": "touched_and_conflicted",
                   "storage": rep.gpu["storage"],
                   "parallelism": (f"sharded x{world}: scan items by agent row block, "
                                   f"{'A as row blocks + AT replicated' if args.placement == 'rows' else 'A + AT replicated'}, "
                                   f"record exchange: {transport}, replicated commit" if sharded else
                                   f"replicas x{world}" if world > 1 else "single"),
                   "l2": "inputs larger than L2 (8*n^2 B fp64 source + A/AT), no flush needed",
                   "step": "device-resident fp64 input -> layout -> dgs_parallel (trace on) -> sigma/tau on host"},
        "e2e": e2e, "gpu_launches": int(launches), "roofline": roofline, "cpu_baseline": cpu,
        "clocks": clocks,
        "solve": {"objective": rep.assignment.value, "outer_iterations": rep.outer_iterations,
                  "inner_iterations": rep.gpu["inner_iterations"], "switches": rep.switches_applied,
                  "pair_items": rep.gpu["pair_items"], "lfmm_rounds": rep.gpu["lfmm_rounds"],
                  "bytes_scanned": rep.gpu["bytes_scanned"], "solve_ms_internal": rep.elapsed / 1e6,
                  "trace_len": rep.gpu["trace_len"]},
        "step_ms_all": times,
        "greedy_start": greedy,
        "sharded": blocks,
    }
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--replicas", action="store_true", help="N > 1: independent instances instead of one sharded solve")
    ap.add_argument("--exchange", default="p2p", choices=["p2p", "nccl"],
                    help="N > 1 sharded: record exchange over peer memory (default) or an NCCL allgather")
    ap.add_argument("--placement", default="rows", choices=["rows", "replicas"],
                    help="N > 1 sharded: each rank holds its row block of A + all of AT (rows), or full replicas")
    ap.add_argument("--blocks", default="c4,c5",
                    help="comma list of BASELINE configs to also run sharded at this N (\"\" for none)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="N > 1 process-group backend (gloo: ranks sharing one GPU, for tests)")
    args = ap.parse_args()
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference(args, wl)
    else:
        run_ours(args, wl)


if __name__ == "__main__":
    main()
