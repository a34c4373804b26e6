"""Host-side mirror of the reference's solver interface for the DGS hot path.

Names, argument meaning and error behaviour follow the reference's public C++
API (paths relative to /root/reference/proj):

* data types           include/lsap/types.hpp:31-104, include/lsap/parallel.hpp:12-55
* dgs_parallel         include/lsap/parallel.hpp:80   -> lsapgpu_solve
* evaluate_all_parallel parallel.hpp:60-61            -> lsapgpu_evaluate_all
* check_conflicts      parallel.hpp:65                -> lsapgpu_check_conflicts
* apply_parallel_switches parallel.hpp:71-74          -> lsapgpu_apply_parallel_switches
* random_perm / make_assignment / objective / initial_random
                       include/lsap/rng.hpp:37-46, src/core.cpp:17-50, src/dgs.cpp:22-25

Every compute call goes through the C-ABI of liblsapgpu.so (the sm_100a
kernels).  The only host arithmetic is what the reference also does
sequentially on the host: the Fisher-Yates permutation and the ordered
objective sum.
"""
from __future__ import annotations

import ctypes as C
import sys
import threading
from collections.abc import Sequence
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

from . import _native as N

TRACE_CAP = 100000  # parallel.cpp:15


class Error(RuntimeError):
    """lsap::Error (types.hpp:17-20)."""


class InternalError(Error):
    """The conflict-freeness assertion (parallel.cpp:296-302)."""


# ---------------------------------------------------------------------------
# data model (types.hpp)
# ---------------------------------------------------------------------------
class Instance:
    """Square benefit matrix, row-major fp64 (types.hpp:31-54)."""

    def __init__(self, n: int = 0, benefits=None):
        self.n = int(n)
        if benefits is None:
            benefits = np.zeros(self.n * self.n)
        self.benefits = np.ascontiguousarray(np.asarray(benefits, dtype=np.float64).reshape(-1))

    @classmethod
    def from_matrix(cls, a) -> "Instance":
        a = np.asarray(a, dtype=np.float64)
        return cls(a.shape[0], a)

    @staticmethod
    def zeros(n: int) -> "Instance":
        return Instance(n, np.zeros(n * n))

    def matrix(self) -> np.ndarray:
        return self.benefits.reshape(self.n, self.n)

    def at(self, i: int, j: int) -> float:
        return float(self.benefits[i * self.n + j])

    def row(self, i: int) -> np.ndarray:
        return self.benefits[i * self.n:(i + 1) * self.n]

    def validate(self) -> None:
        """core.cpp:9-15 (the device repeats this check on upload)."""
        if self.n < 1:
            raise Error(f"instance size must be >= 1, got {self.n}")
        if self.benefits.size != self.n * self.n:
            raise Error(f"benefit matrix is not {self.n}x{self.n}")
        if not np.isfinite(self.benefits).all():
            raise Error("benefit matrix contains a non-finite entry")


@dataclass
class Assignment:
    """sigma: job -> agent, tau: agent -> job, value: cached objective (types.hpp:58-64)."""
    sigma: np.ndarray
    tau: np.ndarray
    value: float = 0.0

    def size(self) -> int:
        return len(self.sigma)


@dataclass
class ExchangeRecord:
    partner: int = -1
    delta: float = 0.0
    active: bool = False


class DeltaTables:
    """SoA storage of DeltaTables (types.hpp:74-84): records are views."""

    def __init__(self, n: int = 0):
        self.agent_delta = np.zeros(n)
        self.agent_partner = np.full(n, -1, np.int32)
        self.agent_active = np.zeros(n, np.uint8)
        self.job_delta = np.zeros(n)
        self.job_partner = np.full(n, -1, np.int32)
        self.job_active = np.zeros(n, np.uint8)

    @staticmethod
    def sized(n: int) -> "DeltaTables":
        return DeltaTables(n)

    @property
    def n(self) -> int:
        return len(self.agent_delta)

    def set_agent(self, i: int, rec: ExchangeRecord) -> None:
        self.agent_partner[i], self.agent_delta[i], self.agent_active[i] = rec.partner, rec.delta, rec.active

    def set_job(self, j: int, rec: ExchangeRecord) -> None:
        self.job_partner[j], self.job_delta[j], self.job_active[j] = rec.partner, rec.delta, rec.active

    def agent_record(self, i: int) -> ExchangeRecord:
        return ExchangeRecord(int(self.agent_partner[i]), float(self.agent_delta[i]), bool(self.agent_active[i]))

    def job_record(self, j: int) -> ExchangeRecord:
        return ExchangeRecord(int(self.job_partner[j]), float(self.job_delta[j]), bool(self.job_active[j]))

    def identical(self, other: "DeltaTables") -> bool:
        """test_parallel.cpp:31-43: partner, active and the delta bits."""
        return (np.array_equal(self.agent_partner, other.agent_partner)
                and np.array_equal(self.job_partner, other.job_partner)
                and np.array_equal(self.agent_active, other.agent_active)
                and np.array_equal(self.job_active, other.job_active)
                and np.array_equal(self.agent_delta.view(np.uint64), other.agent_delta.view(np.uint64))
                and np.array_equal(self.job_delta.view(np.uint64), other.job_delta.view(np.uint64)))


@dataclass
class ParallelConfig:
    """ParallelConfig : DgsConfig (parallel.hpp:12-31, dgs.hpp:10-21).

    ``workers`` and ``chunk`` are accepted and validated like the reference's
    but do not change anything (results never depend on them,
    parallel.hpp:79-80).  ``device`` and ``use_graph`` are the GPU additions.
    """
    seed: int = 0
    deadline: Optional[int] = None  # nanoseconds; None = no deadline
    improvement_epsilon: float = 0.0
    workers: int = 0
    chunk: int = 64
    reeval: str = "touched_and_conflicted"  # or "touched_only"
    device: int = 0
    use_graph: bool = True
    init: str = "random"  # extension: "greedy" starts from the device greedy assignment

    def validate(self) -> None:
        if self.init not in ("random", "greedy"):
            raise Error(f"unknown init '{self.init}'")
        if not (self.improvement_epsilon >= 0.0):
            raise Error("improvement_epsilon must be >= 0")
        if self.workers < 0:
            raise Error("workers must be >= 1 (0 = auto)")
        if self.chunk < 1:
            raise Error("chunk must be >= 1")
        if self.reeval not in ("touched_and_conflicted", "touched_only"):
            raise Error(f"unknown reeval policy '{self.reeval}'")


@dataclass
class AuctionConfig:
    """AuctionConfig (baselines.hpp:12-26)."""
    epsilon: Optional[float] = None  # None: (max - min) / (2n), or 1.0 for a constant matrix
    scaling: bool = False
    scale_factor: float = 4.0
    deadline: Optional[int] = None   # nanoseconds; None = no deadline
    device: int = 0

    def validate(self) -> None:
        if self.epsilon is not None and not (self.epsilon > 0.0):
            raise Error("auction: epsilon must be > 0")
        if not (self.scale_factor > 1.0):
            raise Error("auction: scale_factor must be > 1")


@dataclass
class ConflictSets:
    reserved: List[int]
    conflicted: List[int]
    agent_accepted: np.ndarray
    job_accepted: np.ndarray
    conflicted_jobs: List[int]


@dataclass
class AppliedExchange:
    agent: int = -1
    new_job: int = -1
    old_job: int = -1
    displaced: int = -1
    delta: float = 0.0


class ObjectiveTrace(Sequence):
    """SolveReport::objective_trace (types.hpp:97-105): (switches, value)
    pairs, held as the two arrays the library filled and turned into Python
    tuples only when read (a 10^5-entry trace is ~10 ms of tuple building)."""

    __slots__ = ("switches", "values")

    def __init__(self, switches: np.ndarray, values: np.ndarray):
        self.switches = switches
        self.values = values

    def __len__(self) -> int:
        return len(self.switches)

    def __getitem__(self, k):
        if isinstance(k, slice):
            return list(zip(self.switches[k].tolist(), self.values[k].tolist()))
        return (int(self.switches[k]), float(self.values[k]))

    def __iter__(self):
        return iter(zip(self.switches.tolist(), self.values.tolist()))

    def __eq__(self, other) -> bool:
        if isinstance(other, ObjectiveTrace):
            return (np.array_equal(self.switches, other.switches)
                    and np.array_equal(self.values, other.values))
        try:
            other = list(other)
        except TypeError:
            return NotImplemented
        if len(other) != len(self):
            return False
        if not other:
            return True
        sw = np.array([t[0] for t in other], np.int64)
        va = np.array([t[1] for t in other], np.float64)
        return np.array_equal(self.switches, sw) and np.array_equal(self.values, va)

    def __repr__(self) -> str:
        return f"ObjectiveTrace({len(self)} entries)"


@dataclass
class SolveReport:
    assignment: Assignment
    objective_trace: Sequence[Tuple[int, float]] = field(default_factory=list)
    outer_iterations: int = 0
    switches_applied: int = 0
    elapsed: int = 0  # nanoseconds
    terminated_by: str = "converged"
    gap_vs_oracle: Optional[float] = None
    completed_greedily: bool = False
    gpu: dict = field(default_factory=dict)  # GPU instrumentation (lsapgpu_stats)


# ---------------------------------------------------------------------------
# host helpers identical to the reference's
# ---------------------------------------------------------------------------
def random_perm(n: int, seed: int) -> np.ndarray:
    """rng.hpp:37-46."""
    p = np.empty(n, np.int32)
    N.LIB.lsapgpu_random_perm(n, seed & 0xFFFFFFFFFFFFFFFF, N.ptr(p))
    return p


def is_permutation(p) -> bool:
    p = np.asarray(p)
    n = len(p)
    return bool(((p >= 0) & (p < n)).all() and len(np.unique(p)) == n)


def make_tau(sigma) -> np.ndarray:
    sigma = np.asarray(sigma, np.int32)
    if not is_permutation(sigma):
        raise Error("invalid assignment: not a permutation")
    tau = np.empty_like(sigma)
    tau[sigma] = np.arange(len(sigma), dtype=np.int32)
    return tau


def objective(inst: Instance, asg: Assignment) -> float:
    """core.cpp:17-24: sum over jobs in ascending order (sequential fp64)."""
    if asg.size() != inst.n:
        raise Error(f"assignment size {asg.size()} does not match instance size {inst.n}")
    vals = inst.benefits[np.asarray(asg.sigma, np.int64) * inst.n + np.arange(inst.n)]
    return float(np.cumsum(vals)[-1]) if inst.n else 0.0


def make_assignment(inst: Instance, sigma) -> Assignment:
    """core.cpp:44-50."""
    sigma = np.ascontiguousarray(sigma, np.int32)
    asg = Assignment(sigma, make_tau(sigma), 0.0)
    asg.value = objective(inst, asg)
    return asg


def initial_random(inst: Instance, seed: int) -> Assignment:
    """dgs.cpp:22-25."""
    inst.validate()
    return make_assignment(inst, random_perm(inst.n, seed))


def agent_exchange_delta(inst: Instance, asg: Assignment, i: int, j_new: int) -> float:
    """core.hpp:25-31 (for tests / properties)."""
    j_old = int(asg.tau[i])
    d = int(asg.sigma[j_new])
    return (inst.at(i, j_new) - inst.at(i, j_old)) + (inst.at(d, j_old) - inst.at(d, j_new))


# ---------------------------------------------------------------------------
# the device context
# ---------------------------------------------------------------------------
class Context:
    """Owns one lsapgpu_ctx (device memory, stream, cached CUDA graph)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        rc = N.LIB.lsapgpu_create(C.byref(h), device)
        if rc != N.OK:
            raise Error(f"lsapgpu_create failed (rc={rc}): no usable sm_100 CUDA device {device}")
        self.h = h
        self.device = device
        self._trace_pool: list = []

    def _trace_buffers(self, cap: int):
        """Trace output arrays (switches, values) of at least ``cap`` entries.
        A pair is reused once no report still views it: fresh arrays cost a
        page fault per 4 KB the library writes (~0.1 ms for a C3 trace)."""
        for pair in self._trace_pool:
            # 2 = the pool's tuple + getrefcount's argument: no live views
            if pair[0].size >= cap and sys.getrefcount(pair[0]) == 2 and sys.getrefcount(pair[1]) == 2:
                return pair
        pair = (np.empty(max(cap, 1), np.int64), np.empty(max(cap, 1)))
        if len(self._trace_pool) < 4:
            self._trace_pool.append(pair)
        return pair

    def close(self) -> None:
        if getattr(self, "h", None):
            N.LIB.lsapgpu_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int) -> None:
        if rc == N.OK:
            return
        msg = N.LIB.lsapgpu_last_error(self.h).decode()
        if rc == N.ERR_INTERNAL:
            raise InternalError(msg)
        raise Error(msg)

    # -- instance ---------------------------------------------------------
    @property
    def n(self) -> int:
        return int(N.LIB.lsapgpu_n(self.h))

    @property
    def storage(self) -> str:
        return N.STORAGE_NAMES.get(int(N.LIB.lsapgpu_storage(self.h)), "none")

    @property
    def storage_bytes(self) -> int:
        return N.STORAGE_BYTES[int(N.LIB.lsapgpu_storage(self.h))]

    def set_matrix(self, a, n: Optional[int] = None) -> None:
        """Host matrix (numpy, any of f64/f32/i32/i16) or a CUDA torch tensor."""
        if hasattr(a, "is_cuda") and a.is_cuda:
            import torch
            dt = {torch.float64: N.F64, torch.float32: N.F32, torch.int32: N.I32, torch.int16: N.I16}[a.dtype]
            t = a.contiguous()
            nn = int(n if n is not None else t.shape[0])
            self._check(N.LIB.lsapgpu_set_matrix_device(self.h, t.data_ptr(), nn, dt))
            return
        if hasattr(a, "numpy"):
            a = a.numpy()
        a = np.ascontiguousarray(a)
        dt = {np.dtype(np.float64): N.F64, np.dtype(np.float32): N.F32, np.dtype(np.int32): N.I32,
              np.dtype(np.int16): N.I16}.get(a.dtype)
        if dt is None:
            a = a.astype(np.float64)
            dt = N.F64
        nn = int(n if n is not None else (a.shape[0] if a.ndim == 2 else int(round(np.sqrt(a.size)))))
        if nn >= 1 and a.size != nn * nn:
            raise Error(f"benefit matrix is not {nn}x{nn}")
        self._check(N.LIB.lsapgpu_set_matrix(self.h, N.ptr(a), nn, dt))

    def set_instance(self, inst: Instance) -> None:
        """Upload an Instance (no caching: instances are plain mutable arrays,
        so every reference-style call re-uploads; keep a Context and call
        set_matrix once to amortise uploads over many solves)."""
        if inst.n < 1:
            raise Error(f"instance size must be >= 1, got {inst.n}")
        if inst.benefits.size != inst.n * inst.n:
            raise Error(f"benefit matrix is not {inst.n}x{inst.n}")
        self._check(N.LIB.lsapgpu_set_matrix(self.h, N.ptr(inst.benefits), inst.n, N.F64))

    def generate(self, kind: str, n: int, seed: int = 0, param: Optional[float] = None) -> None:
        """On-device synthetic instance: int | f32 | unit | p2p | geom."""
        if param is None:
            param = {"int": 1000.0, "unit": 10.0, "geom": 100.0}.get(kind, 0.0)
        self._check(N.LIB.lsapgpu_generate(self.h, N.GEN[kind], n, seed & 0xFFFFFFFFFFFFFFFF, float(param)))

    def read_rows(self, rows) -> np.ndarray:
        rows = np.ascontiguousarray(rows, np.int32)
        out = np.empty((len(rows), self.n))
        self._check(N.LIB.lsapgpu_read_rows(self.h, N.ptr(rows), len(rows), N.ptr(out)))
        return out

    # -- solver -----------------------------------------------------------
    def solve(self, cfg: ParallelConfig = ParallelConfig(), init_sigma=None, trace: bool = True,
              dist=None):
        """lsap::dgs_parallel on this context's matrix.  ``dist`` (see
        paper_1106_5694_b200.dist) makes it one rank of a multi-GPU solve."""
        cfg.validate()
        n = self.n
        p = N.Params()
        p.seed = cfg.seed & 0xFFFFFFFFFFFFFFFF
        p.eps = cfg.improvement_epsilon
        p.reeval = 0 if cfg.reeval == "touched_and_conflicted" else 1
        p.use_graph = 1 if cfg.use_graph else 0
        # Deadline::starting accepts any budget: zero or negative expires at once
        p.deadline_ns = -1 if cfg.deadline is None else max(0, int(cfg.deadline))
        p.init_mode = 1 if getattr(cfg, "init", "random") == "greedy" else 0
        if init_sigma is not None:
            init_sigma = np.ascontiguousarray(init_sigma, np.int32)
            p.init_sigma = init_sigma.ctypes.data
        sigma = np.empty(n, np.int32)
        tau = np.empty(n, np.int32)
        st = N.Stats()
        cap = TRACE_CAP + 4096 if trace else 0
        ts, tv = self._trace_buffers(cap) if trace else (None, None)
        tl = C.c_int64(0)

        def run():
            if dist is None:
                rc = N.LIB.lsapgpu_solve(self.h, C.byref(p), N.ptr(sigma), N.ptr(tau), C.byref(st),
                                         N.ptr(ts) if trace else None, N.ptr(tv) if trace else None, cap,
                                         C.byref(tl))
            else:
                rc = N.LIB.lsapgpu_solve_dist(self.h, C.byref(p), C.byref(dist.struct(self)), N.ptr(sigma),
                                              N.ptr(tau), C.byref(st), N.ptr(ts) if trace else None,
                                              N.ptr(tv) if trace else None, cap, C.byref(tl))
                dist.raise_pending()
            self._check(rc)

        run()
        if trace and tl.value > cap and cfg.deadline is None and dist is None:
            # the reference's trace grows by one entry per outer pass past its
            # 100000 cap (parallel.cpp:15-20,343-344): re-run with room for all
            # of it (deterministic without a deadline)
            cap = int(tl.value)
            ts, tv = np.empty(cap, np.int64), np.empty(cap)
            run()
        k = min(tl.value, cap)
        rep = SolveReport(
            assignment=Assignment(sigma, tau, st.value),
            objective_trace=ObjectiveTrace(ts[:k], tv[:k]) if trace else [],
            outer_iterations=st.outer_iterations,
            switches_applied=st.switches_applied,
            elapsed=int(st.elapsed_ms * 1e6),
            terminated_by="deadline" if st.terminated_by else "converged",
        )
        rep.gpu = st.as_dict()
        rep.gpu["storage"] = N.STORAGE_NAMES[st.storage]
        rep.gpu["trace_len"] = tl.value
        return rep

    def greedy_assignment(self):
        """Greedy assignment of this context's matrix (extension; see
        lsapgpu_greedy_assignment): (sigma, claim rounds)."""
        sigma = np.empty(self.n, np.int32)
        rounds = C.c_int64(0)
        self._check(N.LIB.lsapgpu_greedy_assignment(self.h, N.ptr(sigma), C.byref(rounds)))
        return sigma, rounds.value

    def auction_solve(self, cfg: Optional["AuctionConfig"] = None, on_round=None,
                      round_cap: int = 4096) -> SolveReport:
        """lsap::auction_solve (auction.cpp:110-153) on this context's matrix.
        ``on_round`` observes the price vector after every round (the device
        records up to ``round_cap`` rounds; without a deadline a longer run is
        repeated with an exact-size buffer, the solve being deterministic)."""
        cfg = cfg or AuctionConfig()
        cfg.validate()
        n = self.n
        p = N.AuctionParams()
        p.has_epsilon = 0 if cfg.epsilon is None else 1
        p.epsilon = 0.0 if cfg.epsilon is None else float(cfg.epsilon)
        p.scaling = 1 if cfg.scaling else 0
        p.scale_factor = float(cfg.scale_factor)
        p.deadline_ns = -1 if cfg.deadline is None else max(0, int(cfg.deadline))
        sigma = np.empty(n, np.int32)
        tau = np.empty(n, np.int32)
        prices = np.empty(n)
        st = N.AuctionStats()

        def run(cap):
            rp = np.empty((cap, n)) if cap else None
            self._check(N.LIB.lsapgpu_auction_solve(self.h, C.byref(p), N.ptr(sigma), N.ptr(tau), C.byref(st),
                                                    N.ptr(prices), N.ptr(rp) if cap else None, cap))
            return rp

        cap = round_cap if on_round is not None else 0
        rp = run(cap)
        if on_round is not None and st.outer_iterations > cap and cfg.deadline is None:
            cap = int(st.outer_iterations)
            rp = run(cap)
        if on_round is not None:
            for r in range(min(cap, st.outer_iterations)):
                on_round(rp[r])
        rep = SolveReport(
            assignment=Assignment(sigma, tau, st.value),
            objective_trace=[(0, st.value)],  # auction.cpp:149
            outer_iterations=st.outer_iterations,
            switches_applied=st.switches_applied,
            elapsed=int(st.elapsed_ms * 1e6),
            terminated_by="deadline" if st.terminated_by else "converged",
            completed_greedily=bool(st.completed_greedily),
        )
        rep.gpu = st.as_dict()
        rep.gpu["storage"] = N.STORAGE_NAMES[st.storage]
        rep.gpu["prices"] = prices
        return rep

    def evaluate_all(self, sigma, eps: float = 0.0) -> DeltaTables:
        sigma = np.ascontiguousarray(sigma, np.int32)
        n = self.n
        t = DeltaTables(n)
        self._check(N.LIB.lsapgpu_evaluate_all(self.h, N.ptr(sigma), float(eps), N.ptr(t.agent_delta),
                                               N.ptr(t.agent_partner), N.ptr(t.job_delta),
                                               N.ptr(t.job_partner)))
        t.agent_active[:] = t.agent_partner >= 0
        t.job_active[:] = t.job_partner >= 0
        return t

    def check_conflicts(self, tables: DeltaTables, sigma) -> ConflictSets:
        sigma = np.ascontiguousarray(sigma, np.int32)
        n = len(sigma)
        if tables.n != n:
            raise Error("delta tables do not match assignment size")
        ad = np.where(tables.agent_active != 0, tables.agent_delta, 0.0)
        jd = np.where(tables.job_active != 0, tables.job_delta, 0.0)
        ap = np.ascontiguousarray(tables.agent_partner, np.int32)
        jp = np.ascontiguousarray(tables.job_partner, np.int32)
        outs = [np.empty(n, np.uint8) for _ in range(4)]
        cj = np.empty(n, np.int32)
        k = C.c_int32(0)
        self._check(N.LIB.lsapgpu_check_conflicts(self.h, n, N.ptr(ad), N.ptr(ap), N.ptr(jd), N.ptr(jp),
                                                  N.ptr(sigma), *[N.ptr(o) for o in outs], N.ptr(cj),
                                                  C.byref(k)))
        return ConflictSets(reserved=np.flatnonzero(outs[2]).tolist(),
                            conflicted=np.flatnonzero(outs[3]).tolist(),
                            agent_accepted=outs[0], job_accepted=outs[1],
                            conflicted_jobs=cj[:k.value].tolist())

    def apply_parallel_switches(self, asg: Assignment, tables: DeltaTables, sets: ConflictSets,
                                eps: float = 0.0):
        n = self.n
        if asg.size() != n:
            raise Error("assignment does not match instance")
        s = np.ascontiguousarray(asg.sigma, np.int32).copy()
        t = np.ascontiguousarray(asg.tau, np.int32).copy()
        v = C.c_double(asg.value)
        outs = [np.empty(n, np.int32) for _ in range(4)] + [np.empty(n)]
        k = C.c_int32(0)
        arrs = [np.ascontiguousarray(x) for x in (
            tables.agent_delta, tables.agent_partner.astype(np.int32), tables.agent_active.astype(np.uint8),
            tables.job_delta, tables.job_partner.astype(np.int32), tables.job_active.astype(np.uint8),
            np.asarray(sets.agent_accepted, np.uint8), np.asarray(sets.job_accepted, np.uint8))]
        self._check(N.LIB.lsapgpu_apply_parallel_switches(
            self.h, N.ptr(s), N.ptr(t), C.byref(v), *[N.ptr(a) for a in arrs], float(eps),
            *[N.ptr(o) for o in outs], C.byref(k)))
        applied = [AppliedExchange(int(outs[0][q]), int(outs[1][q]), int(outs[2][q]), int(outs[3][q]),
                                   float(outs[4][q])) for q in range(k.value)]
        return Assignment(s, t, v.value), applied

    def counters(self) -> dict:
        h, d, k = C.c_int64(), C.c_int64(), C.c_int64()
        self._check(N.LIB.lsapgpu_counters(self.h, C.byref(h), C.byref(d), C.byref(k)))
        return {"h2d_bytes": h.value, "d2h_bytes": d.value, "kernel_launches": k.value}

    @property
    def stream(self) -> int:
        return int(N.LIB.lsapgpu_stream(self.h) or 0)

    def set_timeline(self, capacity: int) -> None:
        """Enable (capacity > 0) or disable the device timeline of scan / commit launches."""
        self._check(N.LIB.lsapgpu_set_timeline(self.h, int(capacity)))

    def timeline(self, capacity: int = 4096):
        """[(t_ns, kind)] since the last call; kind 1 full sweep, 2 scan, 3 commit, 4 commit end."""
        buf = np.zeros(capacity, np.uint64)
        cnt = N.LIB.lsapgpu_timeline(self.h, buf.ctypes.data, capacity)
        return [(int(v >> 4), int(v & 15)) for v in buf[:cnt]]

    def set_scan_timing(self, on: bool) -> None:
        self._check(N.LIB.lsapgpu_set_scan_timing(self.h, 1 if on else 0))

    def scan_timing(self) -> dict:
        tot, fl, cm = C.c_double(), C.c_double(), C.c_double()
        la, fla, cl = C.c_int64(), C.c_int64(), C.c_int64()
        self._check(N.LIB.lsapgpu_scan_timing(self.h, C.byref(tot), C.byref(la), C.byref(fl), C.byref(fla),
                                              C.byref(cm), C.byref(cl)))
        return {"scan_ms": tot.value, "scan_launches": la.value, "full_ms": fl.value,
                "full_launches": fla.value, "commit_ms": cm.value, "commit_launches": cl.value}

    def set_placement(self, rank: int, world: int) -> None:
        """Row-block placement (lsapgpu_set_placement): hold only rank's row
        block of A (plus all of AT) for the multi-GPU solve; set before the
        matrix."""
        self._check(N.LIB.lsapgpu_set_placement(self.h, int(rank), int(world)))

    def scan_plan(self) -> dict:
        """The pair-scan plan chosen for the current matrix (lsapgpu_scan_plan)."""
        info = np.zeros(16, np.int32)
        k = N.LIB.lsapgpu_scan_plan(self.h, N.ptr(info), 16)
        if k < 0:
            self._check(k)
        names = ["kernel", "m", "bufs", "filter", "ctas", "threads", "smem", "chunk", "filter_queue", "filter_tmem"]
        out = dict(zip(names, info[:k].tolist()))
        out["kernel"] = ["streaming", "resident", "filter"][out["kernel"]]
        return out


_ctx_lock = threading.Lock()
_contexts: dict = {}


def generate_instance(kind: str, n: int, seed: int = 0, param: Optional[float] = None,
                      device: int = 0) -> np.ndarray:
    """Synthetic instance (SURVEY 8(d) recipes) built by the on-device generator
    and returned as the reference's host fp64 row-major matrix (n x n)."""
    ctx = Context(device)
    try:
        ctx.generate(kind, n, seed, param)
        return ctx.read_rows(np.arange(n, dtype=np.int32))
    finally:
        ctx.close()


def context(device: int = 0) -> Context:
    """Default context per (host thread, device), like the C++ wrapper's
    thread_local contexts: ctypes releases the GIL inside the library, so
    threads sharing one context would interleave set_instance and solve.
    The reference lets distinct solves run concurrently; so does this."""
    key = (threading.get_ident(), device)
    with _ctx_lock:
        c = _contexts.get(key)
        if c is None:
            c = _contexts[key] = Context(device)
        return c


# ---------------------------------------------------------------------------
# the reference's entry points
# ---------------------------------------------------------------------------
def dgs_parallel(inst: Instance, cfg: Optional[ParallelConfig] = None) -> SolveReport:
    """lsap::dgs_parallel (parallel.hpp:80) on the B200."""
    cfg = cfg or ParallelConfig()
    ctx = context(cfg.device)
    ctx.set_instance(inst)  # Instance::validate (core.cpp:9-15) runs on the device
    cfg.validate()
    return ctx.solve(cfg)


def auction_solve(inst: Instance, cfg: Optional[AuctionConfig] = None, on_round=None) -> SolveReport:
    """lsap::auction_solve (baselines.hpp:33-36) on the B200."""
    cfg = cfg or AuctionConfig()
    ctx = context(cfg.device)
    ctx.set_instance(inst)  # Instance::validate on the device
    cfg.validate()
    return ctx.auction_solve(cfg, on_round=on_round)


def evaluate_all_parallel(inst: Instance, asg: Assignment, tables: DeltaTables,
                          cfg: Optional[ParallelConfig] = None) -> None:
    """lsap::evaluate_all_parallel (parallel.hpp:60-61): fills ``tables`` in place."""
    cfg = cfg or ParallelConfig()
    ctx = context(cfg.device)
    ctx.set_instance(inst)  # Instance::validate on the device
    cfg.validate()
    if asg.size() != inst.n:
        raise Error("assignment does not match instance")
    t = ctx.evaluate_all(asg.sigma, cfg.improvement_epsilon)
    tables.__dict__.update(t.__dict__)


def check_conflicts(tables: DeltaTables, asg: Assignment, device: int = 0) -> ConflictSets:
    """lsap::check_conflicts (parallel.hpp:65)."""
    if tables.n != asg.size():
        raise Error("delta tables do not match assignment size")
    return context(device).check_conflicts(tables, asg.sigma)


def apply_parallel_switches(inst: Instance, asg: Assignment, tables: DeltaTables, sets: ConflictSets,
                            cfg: Optional[ParallelConfig] = None):
    """lsap::apply_parallel_switches (parallel.hpp:71-74) -> (Assignment, [AppliedExchange])."""
    cfg = cfg or ParallelConfig()
    ctx = context(cfg.device)
    ctx.set_instance(inst)  # Instance::validate on the device
    cfg.validate()
    if asg.size() != inst.n:
        raise Error("assignment does not match instance")
    return ctx.apply_parallel_switches(asg, tables, sets, cfg.improvement_epsilon)
