"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

    python tests/golden/make_golden.py          (needs oracle/_ref/liblsap_ref.so)

Every value here comes from the unmodified reference library
(oracle/_ref/liblsap_ref.so, built from /root/reference/proj/src by
oracle/Makefile).  Instances are generated with the reference's own splitmix64
stream recipes (rng.hpp:11-46) via the oracle generators, which
test_oracle.py pins against the reference's generate_geom / random_perm.

Outputs:
  golden.json       solve summaries (sigma/tau/trace sha256, value bits,
                    outer iterations, switches) for the BASELINE configs and the
                    reference tests' instances, plus small step-API cases
  small_cases.npz   full sigma / trace / tables for the small cases
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle, RefLib  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def trace_sha(trace) -> str:
    sw = np.array([t[0] for t in trace], np.int64)
    va = np.array([t[1] for t in trace], np.float64)
    return hashlib.sha256(sw.tobytes() + va.tobytes()).hexdigest()


# (name, generator kind, n, instance seed, param, solver seed, policy, eps)
SOLVES = [
    ("c1_int1000", "int", 1000, 0, 1000.0, 0, 0, 0.0),
    ("c2_int5000", "int", 5000, 0, 1000.0, 0, 0, 0.0),
    ("c3_p2p10000", "p2p", 10000, 0, None, 0, 0, 0.0),
    ("int10000", "int", 10000, 0, 1000.0, 0, 0, 0.0),
    ("f32_10000", "f32", 10000, 0, None, 0, 0, 0.0),
    ("c4_f32_30000", "f32", 30000, 0, None, 0, 0, 0.0),
    ("c2_int5000_touched_only", "int", 5000, 0, 1000.0, 0, 1, 0.0),
    ("geom2048_touched_only", "geom", 2048, "derive:13:2048:0", 100.0, 2, 1, 0.0),
    ("geom2048", "geom", 2048, "derive:13:2048:0", 100.0, 2, 0, 0.0),
    ("geom4096_seed2", "geom", 4096, "derive:13:4096:0", 100.0, 2, 0, 0.0),
    ("unit3000_eps", "unit", 3000, 77, 10.0, 5, 0, 0.05),
]
# small cases stored in full: reference test instances
SMALL = [
    ("geom64_w", "geom", 64, 47 + 64, 100.0, 12, 0, 0.0),      # test_parallel.cpp:222-237
    ("geom128_w", "geom", 128, 47 + 128, 100.0, 12, 0, 0.0),
    ("geom48_fp", "geom", 48, 59, 100.0, 4, 0, 0.0),           # test_parallel.cpp:239-256
    ("geom48_fp_touched", "geom", 48, 59, 100.0, 4, 1, 0.0),
    ("geom96_trace", "geom", 96, 61, 100.0, 21, 0, 0.0),       # test_parallel.cpp:258-271
    ("acc_geom64", "geom", 64, "derive:7:64:0", 100.0, 5, 0, 0.0),     # acceptance.cpp:133-159
    ("acc_geom256", "geom", 256, "derive:7:256:0", 100.0, 5, 0, 0.0),
    ("acc_geom1024", "geom", 1024, "derive:7:1024:0", 100.0, 5, 0, 0.0),
    ("geom256_seed2", "geom", 256, 67, 100.0, 2, 0, 0.0),      # test_parallel.cpp:273-283
    ("two_perm", "explicit2", 2, 0, None, 3, 0, 0.0),          # test_parallel.cpp:196-206
] + [("rand_small_%d" % s, "unit", 3 + s % 5, 9500 + s, 10.0, s + 1, 0, 0.0) for s in range(12)]


def resolve_seed(o, seed):
    if isinstance(seed, str) and seed.startswith("derive:"):
        _, base, n, idx = seed.split(":")
        return o.derive_instance_seed(int(base), int(n), int(idx))
    return seed


def instance(o, kind, n, seed, param):
    if kind == "explicit2":
        return np.array([[0.0, 10.0], [10.0, 0.0]])
    return o.generate(kind, n, resolve_seed(o, seed), param)


def main():
    o, r = Oracle(), RefLib()
    out = {"generator": "tests/golden/make_golden.py", "reference_kernel": r.kernel_name(),
           "solves": {}, "small": {}, "perm": {}, "geom_sha": {}, "gen_sha": {}}
    arrays = {}
    for seed in (0, 1, 2, 12345):
        for n in (1, 2, 10, 1000):
            out["perm"][f"{n}:{seed}"] = r.random_perm(n, seed).tolist() if n <= 10 else sha(r.random_perm(n, seed))
    for n, seed in ((64, 111), (300, 5)):
        out["geom_sha"][f"{n}:{seed}"] = sha(r.generate_geom(n, seed))
    for kind, n, seed, param in (("int", 300, 3, 1000.0), ("f32", 300, 4, None), ("unit", 300, 5, 10.0),
                                 ("p2p", 300, 6, None), ("geom", 300, 7, 100.0)):
        out["gen_sha"][f"{kind}:{n}:{seed}"] = sha(o.generate(kind, n, seed, param))

    for name, kind, n, seed, param, run, policy, eps in SOLVES + SMALL:
        a = instance(o, kind, n, seed, param)
        t0 = time.time()
        rep = r.dgs_parallel(a, seed=run, eps=eps, policy=policy, workers=os.cpu_count() or 8)
        rec = {"kind": kind, "n": n, "instance_seed": resolve_seed(o, seed), "param": param, "seed": run,
               "policy": policy, "eps": eps, "sigma_sha": sha(rep.sigma), "tau_sha": sha(rep.tau),
               "value": rep.value, "value_hex": float(rep.value).hex(), "outer": rep.outer_iterations,
               "switches": rep.switches_applied, "terminated_by": rep.terminated_by,
               "trace_len": len(rep.trace), "trace_sha": trace_sha(rep.trace),
               "ref_elapsed_ms": rep.elapsed_ms}
        if (name, kind, n, seed, param, run, policy, eps) in SMALL:
            out["small"][name] = rec
            arrays[name + "__sigma"] = rep.sigma
            arrays[name + "__trace_sw"] = np.array([t[0] for t in rep.trace], np.int64)
            arrays[name + "__trace_v"] = np.array([t[1] for t in rep.trace], np.float64)
        else:
            out["solves"][name] = rec
        print(f"{name:28s} n={n:6d} value={rep.value!r} outer={rep.outer_iterations} "
              f"switches={rep.switches_applied} ({time.time() - t0:.1f}s)", flush=True)

    # step APIs on small instances: evaluate_all tables, check_conflicts, apply
    steps = {}
    for k, (kind, n, seed, sseed) in enumerate([("unit", 37, 801, 3), ("int", 200, 5, 7), ("geom", 150, 41, 3),
                                                 ("f32", 120, 9, 1)]):
        a = o.generate(kind, n, seed)
        sigma = r.random_perm(n, sseed)
        ad, ap, jd, jp = r.evaluate_all(a, sigma)
        cc = r.check_conflicts(ad, ap, jd, jp, sigma)
        tau = np.empty(n, np.int32)
        tau[sigma] = np.arange(n)
        s1, t1, v1, app = r.apply_parallel_switches(
            a, sigma, tau, float(np.cumsum(a[sigma, np.arange(n)])[-1]),
            (ad, ap, (ap >= 0).astype(np.uint8), jd, jp, (jp >= 0).astype(np.uint8)),
            cc["agent_accepted"], cc["job_accepted"])
        key = f"step{k}"
        steps[key] = {"kind": kind, "n": n, "seed": seed, "sigma_seed": sseed, "applied": len(app),
                      "value_after_hex": float(v1).hex()}
        arrays.update({key + "__ad": ad, key + "__ap": ap, key + "__jd": jd, key + "__jp": jp,
                       key + "__acc_a": cc["agent_accepted"], key + "__acc_j": cc["job_accepted"],
                       key + "__reserved": cc["reserved"], key + "__conflicted": cc["conflicted"],
                       key + "__cjobs": cc["conflicted_jobs"], key + "__sigma_after": s1,
                       key + "__applied": np.array([x[:4] for x in app], np.int32).reshape(-1, 4),
                       key + "__applied_delta": np.array([x[4] for x in app], np.float64)})
    out["steps"] = steps
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **arrays)
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
