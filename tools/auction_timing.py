"""Auction baseline timing on the device (SolveReport.elapsed, min of runs)
against the reference's single-threaded time recorded in the golden file.

    python tools/auction_timing.py [case ...]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1106_5694_b200 as g

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
gold = json.load(open(os.path.join(ROOT, "tests", "golden", "auction.json")))["cases"]
names = sys.argv[1:] or ["c1_int1000", "c1_int1000_scaling", "c2_int5000", "c2_int5000_scaling", "p2p1000",
                         "c3_p2p10000", "f32_1000", "geom1024", "geom1024_scaling"]
ctx = g.Context(0)
for nm in names:
    rec = gold[nm]
    seed = rec["instance_seed"]
    if isinstance(seed, str):
        from oracle.oracle import Oracle
        _, b, n, i = seed.split(":")
        seed = Oracle().derive_instance_seed(int(b), int(n), int(i))
    ctx.generate(rec["kind"], rec["n"], seed, rec["param"])
    c = rec["config"]
    cfg = g.AuctionConfig(epsilon=c.get("epsilon"), scaling=c.get("scaling", False),
                          scale_factor=c.get("scale_factor", 4.0))
    ts = []
    for _ in range(3):
        r = ctx.auction_solve(cfg)
        ts.append(r.elapsed / 1e6)
    ok = r.outer_iterations == rec["rounds"] and float(r.assignment.value).hex() == rec["value_hex"]
    print(f"{nm:22s} n={rec['n']:6d} rounds={r.outer_iterations:6d} gpu={min(ts):9.2f} ms "
          f"ref={rec['ref_elapsed_ms']:9.1f} ms  x{rec['ref_elapsed_ms'] / min(ts):7.1f}  "
          f"us/round={1e3 * min(ts) / max(1, r.outer_iterations):6.2f}  match={ok}", flush=True)
