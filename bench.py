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
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
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


def ncu_traffic() -> dict | None:
    """dram bytes per launch of the pair-scan kernel from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_pair_scan_summary.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        return json.load(f)


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
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:  # gloo: several ranks sharing one GPU (tests of the sharded path)
            dist.init_process_group("gloo")
    torch.cuda.set_device(local)
    import paper_1106_5694_b200 as g

    kind, n, iseed, param, desc = wl
    # N > 1: by default ONE instance is solved by all ranks (the sharded solve
    # of DESIGN.md §7: scan items owned by agent index, per-batch record
    # allgather, replicated commit); --replicas: every rank solves its own
    # instance (seed offset by rank)
    sharded = world > 1 and not args.replicas
    if world > 1 and not sharded:
        iseed = iseed + rank
    ctx = g.Context(local)
    cfg = g.ParallelConfig(seed=0)
    stream = torch.cuda.ExternalStream(ctx.stream)
    exch = None
    transport = None

    def solve():
        return ctx.solve(cfg, trace=False, dist=exch)

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
        from paper_1106_5694_b200.dist import TorchDistExchange, TorchPeerExchange
        if a_dev is not None:
            ctx.set_matrix(a_dev)  # exchange buffers are sized for n
        if args.exchange == "p2p":
            # peer-memory transport: the pack kernel stores the records into
            # every replica over NVLink (CUDA IPC mappings); NCCL if it cannot
            # be set up on this node
            try:
                exch = TorchPeerExchange()
                exch.struct(ctx)
                transport = "peer-memory push (pack + allgather in one kernel, CUDA IPC over NVLink)"
            except Exception as e:  # noqa: BLE001
                exch = None
                transport = f"nccl (peer transport unavailable: {e})"
        if exch is None:
            exch = TorchDistExchange()
            transport = transport or f"{args.backend} allgather"

    def step_device():
        ctx.set_matrix(a_dev)
        return solve()

    def step_e2e():
        ctx.set_matrix(a_host.numpy())
        return solve()

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def timed(step, k):
        times = []
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        rep = None
        for _ in range(k):
            barrier()
            ev0.record(stream)
            rep = step()
            ev1.record(stream)
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
    ms = statistics.mean(times)
    if world > 1:
        t = torch.tensor([ms], device=f"cuda:{local}" if args.backend == "nccl" else "cpu")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    launches = (c1["kernel_launches"] - c0["kernel_launches"]) // max(args.steps, 1)

    # e2e through the public API from pinned host memory
    e2e = None
    if a_host is not None:
        for _ in range(max(1, args.warmup // 2)):
            step_e2e()
        e0 = ctx.counters()
        etimes, erep = timed(step_e2e, args.steps)
        e1 = ctx.counters()
        e2e_ms = statistics.mean(etimes)
        if world > 1:
            t = torch.tensor([e2e_ms], device=f"cuda:{local}" if args.backend == "nccl" else "cpu")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": e2e_ms, "unit": "ms",
               "h2d_bytes_per_step": (e1["h2d_bytes"] - e0["h2d_bytes"]) // args.steps,
               "d2h_bytes_per_step": (e1["d2h_bytes"] - e0["d2h_bytes"]) // args.steps,
               "source": "pinned host fp64 (the caller's buffer, DMA'd directly)"}
        # the same call from pageable memory (a plain std::vector / numpy
        # Instance, what a drop-in caller of the C++ API passes): staged
        # through the pinned ring by the host copy threads
        a_pageable = a_host.numpy().copy()

        def step_pageable():
            ctx.set_matrix(a_pageable)
            return solve()

        step_pageable()
        ptimes, _ = timed(step_pageable, max(1, min(args.steps, 5)))
        e2e["pageable_ms"] = statistics.mean(ptimes)

    # roofline of the dominant kernel (pair scan): instrumented host-stepped solve,
    # every scan launch bracketed by CUDA events on the solver's stream
    ctx.set_scan_timing(True)
    trep = ctx.solve(g.ParallelConfig(seed=0, use_graph=False), trace=False)
    ctx.set_scan_timing(False)
    tm = ctx.scan_timing()
    eb = ctx.storage_bytes
    pk = measured_peaks()
    full_bytes = n * 2 * n * eb
    scan_bytes = trep.gpu["bytes_scanned"]
    achieved_all = scan_bytes / (tm["scan_ms"] * 1e-3) / 1e9 if tm["scan_ms"] > 0 else None
    achieved_full = (full_bytes * tm["full_launches"]) / (tm["full_ms"] * 1e-3) / 1e9 if tm["full_ms"] > 0 else None
    tr = ncu_traffic()
    roofline = {
        "bound": "hbm", "achieved": achieved_all, "peak": pk["hbm_gbs"], "unit": "GB/s",
        "frac": achieved_all / pk["hbm_gbs"] if achieved_all else None,
        "traffic": tr.get("dram_bytes_per_launch") if tr else None,
        "kernel": "pair_scan_kernel (all launches of one solve: full sweeps + re-evaluation lists)",
        "algorithmic_bytes_per_launch": scan_bytes / max(tm["scan_launches"], 1),
        "avg_launch_ms": tm["scan_ms"] / max(tm["scan_launches"], 1),
        "full_sweep": {"achieved": achieved_full, "frac": achieved_full / pk["hbm_gbs"] if achieved_full else None,
                       "bytes_per_launch": full_bytes, "avg_launch_ms": tm["full_ms"] / max(tm["full_launches"], 1)},
        "scan_share_of_solve": tm["scan_ms"] / trep.elapsed * 1e6 if trep.elapsed else None,
        "peak_source": pk["source"],
        "traffic_source": tr.get("source") if tr else None,
    }

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
            return ctx.solve(gcfg, trace=False)

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
    out = {
        "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
        "scaling": "strong" if sharded else "weak",
        "vs_baseline": None, "dtype": {"int16": "i16->i32", "int32": "i32", "fp32": "f32->f64",
                                       "fp64": "f64"}[ctx.storage],
        "data": "synthetic",
        "config": {"workload": desc, "n": n, "solver_seed": 0, "reeval": "touched_and_conflicted",
                   "storage": ctx.storage,
                   "parallelism": (f"sharded x{world}: scan items by agent index, record exchange: {transport}, "
                                   f"replicated commit" if sharded else
                                   f"replicas x{world}" if world > 1 else "single"),
                   "l2": "inputs larger than L2 (8*n^2 B fp64 source + A/AT), no flush needed",
                   "step": "device-resident fp64 input -> layout -> dgs_parallel -> sigma/tau on host"},
        "e2e": e2e, "gpu_launches": int(launches), "roofline": roofline, "cpu_baseline": cpu,
        "clocks": clocks,
        "solve": {"objective": rep.assignment.value, "outer_iterations": rep.outer_iterations,
                  "inner_iterations": rep.gpu["inner_iterations"], "switches": rep.switches_applied,
                  "pair_items": rep.gpu["pair_items"], "lfmm_rounds": rep.gpu["lfmm_rounds"],
                  "bytes_scanned": rep.gpu["bytes_scanned"], "solve_ms_internal": rep.elapsed / 1e6},
        "step_ms_all": times,
        "greedy_start": greedy,
    }
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    ctx.close()


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
