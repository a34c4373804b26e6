"""GPU suite for the auction baseline (lsap::auction_solve, auction.cpp:110-153;
SURVEY 8(f) item 4) against the fixtures the reference itself produced
(tests/golden/make_golden_auction.py) and the oracle restatement: sigma, the
value bits, the round and award counts and the final price vector must be
identical; plus the reference's own auction test properties
(test_baselines.cpp:62-160)."""
import hashlib
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "auction.json")))["cases"]
ARR = np.load(os.path.join(HERE, "golden", "auction_small.npz"))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def load(ctx, oracle, rec):
    if rec["kind"] == "explicit2":
        ctx.set_matrix(np.array([[0.0, 10.0], [10.0, 0.0]]))
    elif rec["kind"] == "explicit1":
        ctx.set_matrix(np.array([[4.2]]))
    else:
        seed = rec["instance_seed"]
        if isinstance(seed, str):
            _, base, n, idx = seed.split(":")
            seed = oracle.derive_instance_seed(int(base), int(n), int(idx))
        ctx.generate(rec["kind"], rec["n"], seed, rec["param"])


def acfg(rec):
    import paper_1106_5694_b200 as g
    c = dict(rec["config"])
    return g.AuctionConfig(epsilon=c.get("epsilon"), scaling=c.get("scaling", False),
                           scale_factor=c.get("scale_factor", 4.0), deadline=c.get("deadline_ns"))


@pytest.mark.parametrize("name", sorted(GOLD))
def test_auction_bit_exact_vs_reference(oracle, gpu_ctx, name):
    rec = GOLD[name]
    load(gpu_ctx, oracle, rec)
    rep = gpu_ctx.auction_solve(acfg(rec))
    assert sha(rep.assignment.sigma) == rec["sigma_sha"]
    assert float(rep.assignment.value).hex() == rec["value_hex"]
    assert rep.outer_iterations == rec["rounds"]
    assert rep.switches_applied == rec["switches"]
    assert rep.terminated_by == rec["terminated_by"]
    assert rep.completed_greedily == rec["completed_greedily"]
    assert sha(rep.gpu["prices"]) == rec["prices_sha"]
    tau = np.empty_like(rep.assignment.sigma)
    tau[rep.assignment.sigma] = np.arange(rec["n"], dtype=np.int32)
    assert (rep.assignment.tau == tau).all()


@pytest.mark.parametrize("kind,n,seed,param,cfg", [
    ("int", 500, 11, 100000.0, {}),                      # int32 storage
    ("int", 700, 12, 1000.0, {"scaling": True}),         # int16 storage
    ("unit", 600, 13, 10.0, {"epsilon": 0.01}),          # fp64 storage
    ("f32", 800, 14, None, {"scaling": True, "scale_factor": 3.0}),
    ("geom", 300, 15, 100.0, {}),
    ("p2p", 1500, 16, None, {}),
])
def test_auction_matches_oracle(oracle, gpu_ctx, kind, n, seed, param, cfg):
    import paper_1106_5694_b200 as g
    a = oracle.generate(kind, n, seed, param)
    gpu_ctx.set_matrix(a)
    rep = gpu_ctx.auction_solve(g.AuctionConfig(**cfg))
    want = oracle.auction_solve(a, **cfg)
    assert (rep.assignment.sigma == want.sigma).all()
    assert rep.assignment.value == want.value
    assert rep.outer_iterations == want.rounds
    assert rep.switches_applied == want.switches
    assert rep.gpu["bids"] == want.bids
    assert (rep.gpu["prices"].view(np.int64) == want.prices.view(np.int64)).all()


def test_auction_prices_non_decreasing_every_round(oracle, gpu_ctx):
    """test_baselines.cpp:104-115, through the on_round observer."""
    import paper_1106_5694_b200 as g
    rec = GOLD["geom24_s17"]
    load(gpu_ctx, oracle, rec)
    seen = []
    rep = gpu_ctx.auction_solve(g.AuctionConfig(), on_round=lambda p: seen.append(p.copy()))
    assert len(seen) == rep.outer_iterations == rec["rounds"]
    for p0, p1 in zip(seen, seen[1:]):
        assert (p1 >= p0).all()
    assert sha(seen[-1]) == rec["prices_sha"]


def test_auction_round_buffer_regrows(oracle, gpu_ctx):
    import paper_1106_5694_b200 as g
    rec = GOLD["c1_int1000"]
    load(gpu_ctx, oracle, rec)
    seen = []
    gpu_ctx.auction_solve(g.AuctionConfig(), on_round=lambda p: seen.append(p[0]), round_cap=16)
    assert len(seen) == rec["rounds"]


def test_auction_config_validation(gpu_ctx):
    """test_baselines.cpp:145-153."""
    import paper_1106_5694_b200 as g
    inst = g.Instance.zeros(2)
    with pytest.raises(g.Error, match="epsilon must be > 0"):
        g.auction_solve(inst, g.AuctionConfig(epsilon=0.0))
    with pytest.raises(g.Error, match="scale_factor must be > 1"):
        g.auction_solve(inst, g.AuctionConfig(epsilon=0.1, scale_factor=1.0))


def test_auction_module_api_two_perm():
    """test_baselines.cpp:62-70 through the reference-shaped entry point."""
    import paper_1106_5694_b200 as g
    inst = g.Instance(2, [0.0, 10.0, 10.0, 0.0])
    rep = g.auction_solve(inst, g.AuctionConfig(epsilon=0.1))
    assert rep.assignment.sigma.tolist() == [1, 0]
    assert rep.assignment.value == 20.0
    assert rep.terminated_by == "converged"


def test_auction_constant_matrix_uses_unit_epsilon(oracle, gpu_ctx):
    import paper_1106_5694_b200 as g
    a = np.full((64, 64), 3.0)
    gpu_ctx.set_matrix(a)
    rep = gpu_ctx.auction_solve(g.AuctionConfig())
    want = oracle.auction_solve(a)
    assert rep.gpu["epsilon"] == 1.0
    assert (rep.assignment.sigma == want.sigma).all()
    assert rep.outer_iterations == want.rounds


@pytest.mark.parametrize("name", ["c1_int1000", "geom128_s31", "p2p1000_scaling_sf2"])
def test_auction_global_prices_path(oracle, gpu_ctx, name, monkeypatch):
    """Prices read from global memory (the n > 20480 configuration) on small cases."""
    monkeypatch.setenv("LSAPGPU_AUCTION_LOCAL_PRICES", "0")
    rec = GOLD[name]
    load(gpu_ctx, oracle, rec)
    rep = gpu_ctx.auction_solve(acfg(rec))
    assert sha(rep.assignment.sigma) == rec["sigma_sha"]
    assert float(rep.assignment.value).hex() == rec["value_hex"]
    assert rep.outer_iterations == rec["rounds"]
    assert sha(rep.gpu["prices"]) == rec["prices_sha"]


def test_auction_large_n_global_prices(oracle, gpu_ctx):
    """n above the shared-memory price replica: global-price bidding, vs the oracle."""
    import paper_1106_5694_b200 as g
    n = 21000
    gpu_ctx.generate("int", n, 5, 1000.0)
    rep = gpu_ctx.auction_solve(g.AuctionConfig(epsilon=4.0))
    a = oracle.generate("int", n, 5, 1000.0)
    want = oracle.auction_solve(a, epsilon=4.0)
    assert (rep.assignment.sigma == want.sigma).all()
    assert rep.outer_iterations == want.rounds and rep.switches_applied == want.switches


def test_auction_randomised_sweep():
    """tools/fuzz_auction.py: 150 random auction configurations vs the oracle."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "fuzz_auction.py"), "150", "9"],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
