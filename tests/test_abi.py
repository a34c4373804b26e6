"""CPU suite: the C-ABI library (the product) loads and exports exactly what
include/lsapgpu.h declares; host-side helpers behave like the reference's;
without a GPU the library refuses to run instead of falling back to the CPU."""
import ctypes as C
import json
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lsapgpu.h")
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))


def declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(lsapgpu_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    from paper_1106_5694_b200 import _native as N
    names = declared()
    assert len(names) >= 20
    for nm in names:
        assert hasattr(N.LIB, nm), f"{nm} declared in include/lsapgpu.h but not exported"
    assert sorted(N.EXPORTS) == names


def test_library_is_sm100a_only():
    from paper_1106_5694_b200 import _native as N
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out), out


def test_random_perm_is_the_reference_fisher_yates():
    import paper_1106_5694_b200 as g
    for key, want in GOLD["perm"].items():
        n, seed = map(int, key.split(":"))
        got = g.random_perm(n, seed)
        if n <= 10:
            assert got.tolist() == want
        else:
            import hashlib
            assert hashlib.sha256(got.tobytes()).hexdigest() == want


def test_host_mirror_types_and_errors():
    import paper_1106_5694_b200 as g
    inst = g.Instance(3, np.arange(9.0))
    inst.validate()
    asg = g.make_assignment(inst, [2, 0, 1])
    assert asg.tau.tolist() == [1, 2, 0]
    assert asg.value == inst.at(2, 0) + inst.at(0, 1) + inst.at(1, 2)
    assert g.objective(inst, asg) == asg.value
    with pytest.raises(g.Error, match="not a permutation"):
        g.make_tau([0, 0, 1])
    with pytest.raises(g.Error, match="non-finite"):
        g.Instance(2, [0, np.inf, 1, 2]).validate()
    with pytest.raises(g.Error, match="instance size must be >= 1"):
        g.Instance(0, []).validate()
    with pytest.raises(g.Error, match="benefit matrix is not 2x2"):
        g.Instance(2, [1.0, 2.0, 3.0]).validate()
    for bad, msg in ((dict(improvement_epsilon=-1.0), "improvement_epsilon"), (dict(workers=-1), "workers"),
                     (dict(chunk=0), "chunk"), (dict(reeval="sometimes"), "reeval")):
        with pytest.raises(g.Error, match=msg):
            g.ParallelConfig(**bad).validate()


def test_no_cpu_fallback_without_gpu():
    import torch
    import paper_1106_5694_b200 as g
    from paper_1106_5694_b200 import _native as N
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    h = C.c_void_p()
    assert N.LIB.lsapgpu_create(C.byref(h), 0) == N.ERR_CUDA
    with pytest.raises(g.Error, match="no usable sm_100"):
        g.dgs_parallel(g.Instance(2, [0, 1, 1, 0]))
