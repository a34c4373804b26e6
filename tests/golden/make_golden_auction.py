"""Generate tests/golden/auction.json (+ auction_small.npz) from the REFERENCE.

    python tests/golden/make_golden_auction.py    (needs oracle/_ref/liblsap_ref.so)

Every value comes from the unmodified reference's lsap::auction_solve
(proj/src/auction.cpp:110-153) run through oracle/_ref/liblsap_ref.so; the
instances use the reference's own generator recipes (see make_golden.py).
Cases: the reference's auction tests (test_baselines.cpp:62-160) and the
BASELINE configs C1-C3 under the default, explicit-epsilon and scaling
configurations.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Oracle, RefLib  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# (name, kind, n, instance seed, param, config)
CASES = [
    ("two_perm", "explicit2", 2, 0, None, {"epsilon": 0.1}),               # test_baselines.cpp:62-70
    ("n1", "explicit1", 1, 0, None, {}),                                   # :72-78
    ("geom24_s17", "geom", 24, 17, 100.0, {}),                             # :104-115 (monotone prices)
    ("geom48_s23_scaling", "geom", 48, 23, 100.0, {"scaling": True}),      # :117-133
    ("geom256_s5_deadline0", "geom", 256, 5, 100.0, {"deadline_ns": 0}),   # :135-143
    ("geom128_s31", "geom", 128, 31, 100.0, {}),                           # :155-160
    ("geom1024", "geom", 1024, "derive:13:1024:0", 100.0, {}),
    ("geom1024_scaling", "geom", 1024, "derive:13:1024:0", 100.0, {"scaling": True}),
    ("c1_int1000", "int", 1000, 0, 1000.0, {}),
    ("c1_int1000_scaling", "int", 1000, 0, 1000.0, {"scaling": True}),
    ("c1_int1000_eps", "int", 1000, 0, 1000.0, {"epsilon": 0.25}),
    ("c2_int5000", "int", 5000, 0, 1000.0, {}),
    ("c2_int5000_scaling", "int", 5000, 0, 1000.0, {"scaling": True}),
    ("p2p1000", "p2p", 1000, 0, None, {}),
    ("p2p1000_scaling_sf2", "p2p", 1000, 0, None, {"scaling": True, "scale_factor": 2.0}),
    ("c3_p2p10000", "p2p", 10000, 0, None, {}),
    ("f32_1000", "f32", 1000, 0, None, {}),
    ("unit2000_eps", "unit", 2000, 77, 10.0, {"epsilon": 0.05}),
] + [("int_exact_%d" % s, "int", 2 + s % 6, 4000 + s, 50.0, {"epsilon": 0.9 / (2 + s % 6)})
     for s in range(30)] + [                                               # :80-90
    ("unit_bound_%d" % s, "unit", 2 + s % 7, 6000 + s, 10.0, {"epsilon": 0.05}) for s in range(25)]  # :92-102


def instance(o, kind, n, seed, param):
    if kind == "explicit2":
        return np.array([[0.0, 10.0], [10.0, 0.0]])
    if kind == "explicit1":
        return np.array([[4.2]])
    if isinstance(seed, str):
        _, base, nn, idx = seed.split(":")
        seed = o.derive_instance_seed(int(base), int(nn), int(idx))
    return o.generate(kind, n, seed, param)


def main():
    o, r = Oracle(), RefLib()
    out, arrays = {"generator": "tests/golden/make_golden_auction.py", "cases": {}}, {}
    for name, kind, n, seed, param, cfg in CASES:
        a = instance(o, kind, n, seed, param)
        t0 = time.time()
        rep = r.auction_solve(a, **cfg)
        out["cases"][name] = {
            "kind": kind, "n": n, "instance_seed": seed, "param": param, "config": cfg,
            "sigma_sha": sha(rep.sigma), "prices_sha": sha(rep.prices), "value": rep.value,
            "value_hex": float(rep.value).hex(), "rounds": rep.rounds, "switches": rep.switches,
            "terminated_by": rep.terminated_by, "completed_greedily": rep.completed_greedily,
            "monotone": rep.monotone, "ref_elapsed_ms": rep.elapsed_ms}
        if n <= 1024:
            arrays[name + "__sigma"] = rep.sigma
            arrays[name + "__prices"] = rep.prices
        print(f"{name:26s} n={n:6d} value={rep.value!r} rounds={rep.rounds} switches={rep.switches} "
              f"({time.time() - t0:.1f}s)", flush=True)
    with open(os.path.join(HERE, "auction.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "auction_small.npz"), **arrays)


if __name__ == "__main__":
    main()
