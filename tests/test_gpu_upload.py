"""GPU: the host upload narrows the fp64 matrix on the host before PCIe.

The storage type is speculated from the first 64 rows on the host, every
chunk is converted exactly (int16 / int32 / fp32) by the copy threads, and a
value that does not fit sends the whole upload down the fp64 path again.
Whatever the path, the device layout (hence every result) must equal the one
built from the same matrix already in device memory, and Instance::validate's
error (core.cpp:9-15) must still fire for a non-finite entry anywhere."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _layout_and_solve(ctx, a):
    import paper_1106_5694_b200 as g
    ctx.set_matrix(a)
    rows = ctx.read_rows(np.arange(a.shape[0]))
    rep = ctx.solve(g.ParallelConfig(seed=3))
    return ctx.storage, rows, rep


@pytest.mark.parametrize("case", ["int16", "int32", "fp32", "fp64", "late_fp32", "late_fp64", "late_int32"])
def test_host_narrowing_matches_device_source(gpu_ctx, oracle, case):
    import torch
    n = 2500
    rng = np.random.default_rng(5)
    if case == "int16":
        a = oracle.generate("int", n, 1)
    elif case == "int32":
        a = rng.integers(-300000, 300000, (n, n)).astype(np.float64)
    elif case == "fp32":
        a = oracle.generate("f32", n, 2)
    elif case == "fp64":
        a = oracle.generate("geom", n, 3)
    else:  # first rows narrower than a later row: host speculation fails -> fp64 path
        a = oracle.generate("int", n, 4)
        late = {"late_fp32": 0.5, "late_fp64": 0.1, "late_int32": 1e6}[case]
        a[n - 7, 11] = late
    want = {"int16": "int16", "int32": "int32", "fp32": "fp32", "fp64": "fp64",
            "late_fp32": "fp32", "late_fp64": "fp64", "late_int32": "int32"}[case]
    s_host, rows_host, rep_host = _layout_and_solve(gpu_ctx, a)               # pageable numpy
    s_pin, rows_pin, rep_pin = _layout_and_solve(gpu_ctx, torch.from_numpy(a).pin_memory().numpy())
    s_dev, rows_dev, rep_dev = _layout_and_solve(gpu_ctx, torch.from_numpy(a).cuda())
    assert s_host == s_pin == s_dev == want
    for rows in (rows_host, rows_pin):
        assert np.array_equal(rows.view(np.uint64), rows_dev.view(np.uint64))
    for rep in (rep_host, rep_pin):
        assert np.array_equal(rep.assignment.sigma, rep_dev.assignment.sigma)
        assert rep.objective_trace == rep_dev.objective_trace


@pytest.mark.parametrize("where", ["probe", "late"])
def test_host_upload_rejects_non_finite(gpu_ctx, oracle, where):
    import paper_1106_5694_b200 as g
    n = 1200
    a = oracle.generate("int", n, 6)
    a[3 if where == "probe" else n - 2, 5] = np.inf
    with pytest.raises(g.Error, match="benefit matrix contains a non-finite entry"):
        gpu_ctx.set_matrix(a)
    a[3 if where == "probe" else n - 2, 5] = np.nan
    with pytest.raises(g.Error, match="benefit matrix contains a non-finite entry"):
        gpu_ctx.set_matrix(a)
