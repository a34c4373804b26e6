"""ctypes bindings for the parity checkers (TEST INFRASTRUCTURE ONLY).

* ``Oracle``  -- oracle/liboracle.so, the C restatement in dgs_oracle.c.
* ``RefLib``  -- oracle/_ref/liblsap_ref.so, the unmodified reference library
  compiled from /root/reference/proj/src by oracle/Makefile (+ ref_harness.cpp).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` leg import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "liblsap_ref.so")
TRACE_CAP = 100000  # parallel.cpp:15

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_lp = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_bp = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")


@dataclass
class SolveResult:
    sigma: np.ndarray
    tau: np.ndarray
    value: float
    outer_iterations: int
    switches_applied: int
    terminated_by: str
    elapsed_ms: float
    trace: list = field(default_factory=list)
    inner_iterations: int = -1
    agent_scans: int = -1
    job_scans: int = -1
    pair_items: int = -1


class _Stats(C.Structure):
    _fields_ = [
        ("outer_iterations", C.c_int64),
        ("inner_iterations", C.c_int64),
        ("switches_applied", C.c_int64),
        ("agent_scans", C.c_int64),
        ("job_scans", C.c_int64),
        ("pair_items", C.c_int64),
        ("terminated_by", C.c_int32),
        ("value", C.c_double),
        ("elapsed_ms", C.c_double),
    ]


class _AuctionStats(C.Structure):
    _fields_ = [("rounds", C.c_int64), ("switches", C.c_int64), ("bids", C.c_int64),
                ("terminated_by", C.c_int32), ("completed_greedily", C.c_int32),
                ("value", C.c_double), ("epsilon", C.c_double)]


@dataclass
class AuctionResult:
    sigma: np.ndarray
    value: float
    rounds: int
    switches: int
    terminated_by: str
    completed_greedily: bool
    prices: np.ndarray
    elapsed_ms: float = -1.0
    bids: int = -1
    monotone: bool = True
    round_count: int = -1


def _as(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


class Oracle:
    """The C restatement (dgs_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.lib = C.CDLL(path)
        L.orc_draw.restype = C.c_uint64
        L.orc_draw.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_mix64.restype = C.c_uint64
        L.orc_mix64.argtypes = [C.c_uint64]
        L.orc_derive_instance_seed.restype = C.c_uint64
        L.orc_derive_instance_seed.argtypes = [C.c_uint64, C.c_int32, C.c_int32]
        L.orc_random_perm.argtypes = [C.c_int32, C.c_uint64, _ip]
        L.orc_gen_uniform_int.argtypes = [_dp, C.c_int32, C.c_uint64, C.c_uint64]
        L.orc_gen_unit_f32.argtypes = [_dp, C.c_int32, C.c_uint64]
        L.orc_gen_unit_scaled.argtypes = [_dp, C.c_int32, C.c_uint64, C.c_double]
        L.orc_gen_p2p.argtypes = [_dp, C.c_int32, C.c_uint64]
        L.orc_gen_geom.argtypes = [_dp, C.c_int32, C.c_uint64, C.c_double]
        L.orc_objective.restype = C.c_double
        L.orc_objective.argtypes = [_dp, C.c_int32, _ip]
        L.orc_evaluate_all.argtypes = [_dp, C.c_int32, _ip, C.c_double, _dp, _ip, _dp, _ip]
        L.orc_check_conflicts.restype = C.c_int32
        L.orc_check_conflicts.argtypes = [C.c_int32, _dp, _ip, _dp, _ip, _ip, _bp, _bp, _bp, _bp, _ip]
        L.orc_apply_parallel_switches.restype = C.c_int32
        L.orc_apply_parallel_switches.argtypes = [
            _dp, C.c_int32, _ip, _ip, C.POINTER(C.c_double), _dp, _ip, _bp, _dp, _ip, _bp, _bp, _bp,
            C.c_double, _ip, _ip, _ip, _ip, _dp]
        L.orc_dgs_parallel.restype = C.c_int
        L.orc_dgs_parallel_from.argtypes = [
            _dp, C.c_int32, _ip, C.c_double, C.c_int, C.c_int64, C.c_int, _ip, _ip, C.POINTER(_Stats),
            _lp, _dp, C.c_int64, C.POINTER(C.c_int64)]
        L.orc_greedy_assignment.restype = C.c_int64
        L.orc_greedy_assignment.argtypes = [_dp, C.c_int32, _ip]
        L.orc_auction_solve.argtypes = [_dp, C.c_int32, C.c_int, C.c_double, C.c_int, C.c_double,
                                        C.c_int64, _ip, _dp, C.POINTER(_AuctionStats)]
        L.orc_dgs_parallel.argtypes = [
            _dp, C.c_int32, C.c_uint64, C.c_double, C.c_int, C.c_int64, C.c_int, _ip, _ip,
            C.POINTER(_Stats), _lp, _dp, C.c_int64, C.POINTER(C.c_int64)]

    # -- rng / generators -------------------------------------------------
    def draw(self, seed: int, k: int) -> int:
        return int(self.lib.orc_draw(seed, k))

    def mix64(self, z: int) -> int:
        return int(self.lib.orc_mix64(z))

    def derive_instance_seed(self, base: int, n: int, idx: int) -> int:
        return int(self.lib.orc_derive_instance_seed(base, n, idx))

    def random_perm(self, n: int, seed: int) -> np.ndarray:
        p = np.empty(n, np.int32)
        self.lib.orc_random_perm(n, seed, p)
        return p

    def generate(self, kind: str, n: int, seed: int = 0, param: float | None = None) -> np.ndarray:
        a = np.empty(n * n, np.float64)
        if kind == "int":
            self.lib.orc_gen_uniform_int(a, n, seed, int(param or 1000))
        elif kind == "f32":
            self.lib.orc_gen_unit_f32(a, n, seed)
        elif kind == "unit":
            self.lib.orc_gen_unit_scaled(a, n, seed, float(10.0 if param is None else param))
        elif kind == "p2p":
            self.lib.orc_gen_p2p(a, n, seed)
        elif kind == "geom":
            self.lib.orc_gen_geom(a, n, seed, float(100.0 if param is None else param))
        else:
            raise ValueError(kind)
        return a.reshape(n, n)

    def objective(self, a: np.ndarray, sigma: np.ndarray) -> float:
        n = a.shape[0]
        return float(self.lib.orc_objective(_as(a, np.float64).ravel(), n, _as(sigma, np.int32)))

    # -- step APIs --------------------------------------------------------
    def evaluate_all(self, a, sigma, eps: float = 0.0):
        a = _as(a, np.float64)
        n = a.shape[0]
        ad, jd = np.empty(n), np.empty(n)
        ap, jp = np.empty(n, np.int32), np.empty(n, np.int32)
        self.lib.orc_evaluate_all(a.ravel(), n, _as(sigma, np.int32), eps, ad, ap, jd, jp)
        return ad, ap, jd, jp

    def check_conflicts(self, agent_delta, agent_partner, job_delta, job_partner, sigma):
        n = len(sigma)
        outs = [np.empty(n, np.uint8) for _ in range(4)]
        cj = np.empty(n, np.int32)
        k = self.lib.orc_check_conflicts(n, _as(agent_delta, np.float64), _as(agent_partner, np.int32),
                                         _as(job_delta, np.float64), _as(job_partner, np.int32),
                                         _as(sigma, np.int32), *outs, cj)
        return {"agent_accepted": outs[0], "job_accepted": outs[1], "reserved": outs[2],
                "conflicted": outs[3], "conflicted_jobs": cj[:k].copy()}

    def apply_parallel_switches(self, a, sigma, tau, value, tables, agent_accepted, job_accepted,
                                eps: float = 0.0):
        a = _as(a, np.float64)
        n = a.shape[0]
        s, t = _as(sigma, np.int32).copy(), _as(tau, np.int32).copy()
        v = C.c_double(value)
        ad, ap, aa, jd, jp, ja = tables
        outs = [np.empty(n, np.int32) for _ in range(4)] + [np.empty(n)]
        k = self.lib.orc_apply_parallel_switches(
            a.ravel(), n, s, t, C.byref(v), _as(ad, np.float64), _as(ap, np.int32), _as(aa, np.uint8),
            _as(jd, np.float64), _as(jp, np.int32), _as(ja, np.uint8), _as(agent_accepted, np.uint8),
            _as(job_accepted, np.uint8), eps, *outs)
        if k < 0:
            raise RuntimeError("internal: conflict check admitted overlapping exchanges")
        applied = [(int(outs[0][q]), int(outs[1][q]), int(outs[2][q]), int(outs[3][q]), float(outs[4][q]))
                   for q in range(k)]
        return s, t, v.value, applied

    def dgs_parallel(self, a, seed: int = 0, eps: float = 0.0, policy: int = 0,
                     deadline_ns: int = -1, threads: int = 0, trace: bool = True) -> SolveResult:
        a = _as(a, np.float64)
        n = a.shape[0]
        sig, tau = np.empty(n, np.int32), np.empty(n, np.int32)
        st = _Stats()
        cap = TRACE_CAP + 64 if trace else 0
        ts, tv = np.empty(max(cap, 1), np.int64), np.empty(max(cap, 1))
        tl = C.c_int64(0)
        rc = self.lib.orc_dgs_parallel(a.ravel(), n, seed, eps, policy, deadline_ns, threads, sig, tau,
                                       C.byref(st), ts, tv, cap, C.byref(tl))
        if rc == 1:
            raise ValueError(f"instance size must be >= 1, got {n}")
        if rc == 2:
            raise ValueError("improvement_epsilon must be >= 0")
        if rc == 3:
            raise ValueError("benefit matrix contains a non-finite entry")
        if rc:
            raise RuntimeError(f"oracle failure rc={rc}")
        tr = [(int(ts[k]), float(tv[k])) for k in range(min(tl.value, cap))] if trace else []
        return SolveResult(sig, tau, st.value, st.outer_iterations, st.switches_applied,
                           "deadline" if st.terminated_by else "converged", st.elapsed_ms, tr,
                           st.inner_iterations, st.agent_scans, st.job_scans, st.pair_items)

    def greedy_assignment(self, a):
        """The device greedy-assignment rule (extension): (sigma, rounds)."""
        a = _as(a, np.float64)
        n = a.shape[0]
        sig = np.empty(n, np.int32)
        rounds = self.lib.orc_greedy_assignment(a.ravel(), n, sig)
        return sig, int(rounds)

    def dgs_parallel_from(self, a, init_sigma, eps: float = 0.0, policy: int = 0, threads: int = 0,
                          trace: bool = True) -> SolveResult:
        """dgs_parallel's loop from a given initial sigma (job -> agent)."""
        a = _as(a, np.float64)
        n = a.shape[0]
        sig, tau = np.empty(n, np.int32), np.empty(n, np.int32)
        st = _Stats()
        cap = TRACE_CAP + 64 if trace else 0
        ts, tv = np.empty(max(cap, 1), np.int64), np.empty(max(cap, 1))
        tl = C.c_int64(0)
        rc = self.lib.orc_dgs_parallel_from(a.ravel(), n, _as(init_sigma, np.int32), eps, policy, -1, threads,
                                            sig, tau, C.byref(st), ts, tv, cap, C.byref(tl))
        if rc:
            raise RuntimeError(f"oracle failure rc={rc}")
        tr = [(int(ts[k]), float(tv[k])) for k in range(min(tl.value, cap))] if trace else []
        return SolveResult(sig, tau, st.value, st.outer_iterations, st.switches_applied,
                           "deadline" if st.terminated_by else "converged", st.elapsed_ms, tr,
                           st.inner_iterations, st.agent_scans, st.job_scans, st.pair_items)

    def auction_solve(self, a, epsilon=None, scaling=False, scale_factor=4.0,
                      expire_round: int = -1) -> AuctionResult:
        """auction.cpp restatement; expire_round = k fires the deadline at the
        (k+1)-th round check (0 = the reference's deadline 0)."""
        a = _as(a, np.float64)
        n = a.shape[0]
        sig, pr = np.empty(n, np.int32), np.empty(n)
        st = _AuctionStats()
        if self.lib.orc_auction_solve(a.ravel(), n, 0 if epsilon is None else 1,
                                      0.0 if epsilon is None else float(epsilon), 1 if scaling else 0,
                                      float(scale_factor), expire_round, sig, pr, C.byref(st)):
            raise ValueError("invalid auction instance / config")
        return AuctionResult(sig, st.value, st.rounds, st.switches,
                             "deadline" if st.terminated_by else "converged", bool(st.completed_greedily),
                             pr, bids=st.bids)


class RefLib:
    """The unmodified reference library (oracle/_ref/liblsap_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where /root/reference exists")
        L = self.lib = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_kernel_name.restype = C.c_char_p
        L.ref_random_perm.argtypes = [C.c_int32, C.c_uint64, _ip]
        L.ref_generate_geom.argtypes = [C.c_int32, C.c_double, C.c_uint64, _dp]
        i64p = C.POINTER(C.c_int64)
        L.ref_dgs_parallel.argtypes = [
            _dp, C.c_int32, C.c_uint64, C.c_double, C.c_int, C.c_int64, C.c_int, _ip, _ip,
            C.POINTER(C.c_double), i64p, i64p, C.POINTER(C.c_int), C.POINTER(C.c_double),
            _lp, _dp, C.c_int64, i64p]
        L.ref_auction_solve.argtypes = [_dp, C.c_int32, C.c_int, C.c_double, C.c_int, C.c_double, C.c_int64,
                                        _ip, C.POINTER(C.c_double), C.POINTER(C.c_int64),
                                        C.POINTER(C.c_int64), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                        C.POINTER(C.c_double), _dp, C.POINTER(C.c_int64), C.POINTER(C.c_int)]
        L.ref_evaluate_all.argtypes = [_dp, C.c_int32, _ip, C.c_double, C.c_int, _dp, _ip, _dp, _ip]
        L.ref_check_conflicts.argtypes = [C.c_int32, _dp, _ip, C.c_void_p, _dp, _ip, C.c_void_p, _ip,
                                          _bp, _bp, _bp, _bp, _ip, C.POINTER(C.c_int32)]
        L.ref_apply_parallel_switches.restype = C.c_int32
        L.ref_apply_parallel_switches.argtypes = [
            _dp, C.c_int32, _ip, _ip, C.POINTER(C.c_double), _dp, _ip, _bp, _dp, _ip, _bp, _bp, _bp,
            C.c_double, _ip, _ip, _ip, _ip, _dp]

    def _err(self):
        return self.lib.ref_last_error().decode()

    def kernel_name(self) -> str:
        return self.lib.ref_kernel_name().decode()

    def random_perm(self, n, seed):
        p = np.empty(n, np.int32)
        self.lib.ref_random_perm(n, seed, p)
        return p

    def generate_geom(self, n, seed, bound=100.0):
        a = np.empty(n * n)
        if self.lib.ref_generate_geom(n, bound, seed, a):
            raise ValueError(self._err())
        return a.reshape(n, n)

    def evaluate_all(self, a, sigma, eps=0.0, workers=0):
        a = _as(a, np.float64)
        n = a.shape[0]
        ad, jd = np.empty(n), np.empty(n)
        ap, jp = np.empty(n, np.int32), np.empty(n, np.int32)
        if self.lib.ref_evaluate_all(a.ravel(), n, _as(sigma, np.int32), eps, workers, ad, ap, jd, jp):
            raise ValueError(self._err())
        return ad, ap, jd, jp

    def check_conflicts(self, agent_delta, agent_partner, job_delta, job_partner, sigma):
        n = len(sigma)
        outs = [np.empty(n, np.uint8) for _ in range(4)]
        cj = np.empty(n, np.int32)
        k = C.c_int32(0)
        if self.lib.ref_check_conflicts(n, _as(agent_delta, np.float64), _as(agent_partner, np.int32), None,
                                        _as(job_delta, np.float64), _as(job_partner, np.int32), None,
                                        _as(sigma, np.int32), *outs, cj, C.byref(k)):
            raise ValueError(self._err())
        return {"agent_accepted": outs[0], "job_accepted": outs[1], "reserved": outs[2],
                "conflicted": outs[3], "conflicted_jobs": cj[:k.value].copy()}

    def apply_parallel_switches(self, a, sigma, tau, value, tables, agent_accepted, job_accepted,
                                eps=0.0):
        a = _as(a, np.float64)
        n = a.shape[0]
        s, t = _as(sigma, np.int32).copy(), _as(tau, np.int32).copy()
        v = C.c_double(value)
        ad, ap, aa, jd, jp, ja = tables
        outs = [np.empty(n, np.int32) for _ in range(4)] + [np.empty(n)]
        k = self.lib.ref_apply_parallel_switches(
            a.ravel(), n, s, t, C.byref(v), _as(ad, np.float64), _as(ap, np.int32), _as(aa, np.uint8),
            _as(jd, np.float64), _as(jp, np.int32), _as(ja, np.uint8), _as(agent_accepted, np.uint8),
            _as(job_accepted, np.uint8), eps, *outs)
        if k < 0:
            raise RuntimeError(self._err())
        applied = [(int(outs[0][q]), int(outs[1][q]), int(outs[2][q]), int(outs[3][q]), float(outs[4][q]))
                   for q in range(k)]
        return s, t, v.value, applied

    def dgs_parallel(self, a, seed=0, eps=0.0, policy=0, deadline_ns=-1, workers=0,
                     trace=True) -> SolveResult:
        a = _as(a, np.float64)
        n = a.shape[0]
        sig, tau = np.empty(n, np.int32), np.empty(n, np.int32)
        val, el = C.c_double(), C.c_double()
        outer, sw, tl = C.c_int64(), C.c_int64(), C.c_int64()
        term = C.c_int()
        cap = TRACE_CAP + 64 if trace else 0
        ts, tv = np.empty(max(cap, 1), np.int64), np.empty(max(cap, 1))
        if self.lib.ref_dgs_parallel(a.ravel(), n, seed, eps, policy, deadline_ns, workers, sig, tau,
                                     C.byref(val), C.byref(outer), C.byref(sw), C.byref(term), C.byref(el),
                                     ts, tv, cap, C.byref(tl)):
            raise ValueError(self._err())
        tr = [(int(ts[k]), float(tv[k])) for k in range(min(tl.value, cap))] if trace else []
        return SolveResult(sig, tau, val.value, outer.value, sw.value,
                           "deadline" if term.value else "converged", el.value, tr)

    def auction_solve(self, a, epsilon=None, scaling=False, scale_factor=4.0,
                      deadline_ns: int = -1) -> AuctionResult:
        """lsap::auction_solve (auction.cpp:110-153), with an on_round observer
        recording the last price vector, the round count and monotonicity."""
        a = _as(a, np.float64)
        n = a.shape[0]
        sig, pr = np.empty(n, np.int32), np.empty(n)
        val, el = C.c_double(), C.c_double()
        outer, sw, rounds = C.c_int64(), C.c_int64(), C.c_int64()
        term, greedy, mono = C.c_int(), C.c_int(), C.c_int()
        if self.lib.ref_auction_solve(a.ravel(), n, 0 if epsilon is None else 1,
                                      0.0 if epsilon is None else float(epsilon), 1 if scaling else 0,
                                      float(scale_factor), deadline_ns, sig, C.byref(val), C.byref(outer),
                                      C.byref(sw), C.byref(term), C.byref(greedy), C.byref(el), pr,
                                      C.byref(rounds), C.byref(mono)):
            raise ValueError(self._err())
        return AuctionResult(sig, val.value, outer.value, sw.value,
                             "deadline" if term.value else "converged", bool(greedy.value), pr,
                             elapsed_ms=el.value, monotone=bool(mono.value), round_count=rounds.value)


def load_ref_or_none():
    try:
        return RefLib()
    except (FileNotFoundError, OSError):
        return None
