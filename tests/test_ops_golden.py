"""Operator layer, estimator transforms and the CLI endpoint against the
reference's own outputs (tests/golden/ops.*, made by make_golden_ops.py).

CPU: the oracle's operator-level functions reproduce every fixture (this
pins the checker one kernel at a time).  GPU: the C-ABI operators of
libtsds.so (include/tsds.h), called directly with device pointers, do too;
so do Downsampler.transform / fit_transform and the CLI endpoint's bytes.
"""

import ctypes
import json
import os
import subprocess
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")


@pytest.fixture(scope="module")
def gold():
    with open(os.path.join(GOLD, "ops.json")) as f:
        cases = json.load(f)
    return cases, np.load(os.path.join(GOLD, "ops.npz"))


# ------------------------------------------------------------------ oracle


def test_oracle_ops_match_reference(oracle, gold):
    c, A = gold
    for case in c["width"]:
        out = np.full(case["n_bins"] + 1, -7, np.int64)
        oracle.fill_width_offsets(A[case["x"]], case["x0"], case["span"], case["n_bins"], case["k0"], case["k1"], out)
        assert np.array_equal(out, A[case["want"]]), case
    for case in c["bins"]:
        w = case["width"]
        nb = A[case["off"]].shape[0] - 1
        idx = np.full(w * nb, -5, np.int64)
        cnt = np.full(nb, -5, np.int64)
        oracle.bins_slots(w, A[case["y"]], A[case["off"]], case["b0"], case["b1"], idx, cnt)
        assert np.array_equal(idx, A[case["idx"]]) and np.array_equal(cnt, A[case["cnt"]]), case
    for case in c["compact"]:
        got = oracle.compact_bins(A[case["idx"]], A[case["cnt"]], case["width"])
        assert np.array_equal(got, A[case["want"]])
    for case in c["lttb"]:
        x = None if case["x"] is None else A[case["x"]]
        assert np.array_equal(oracle.lttb_walk(x, A[case["y"]], A[case["off"]]), A[case["want"]])
    for case in c["uniform"]:
        assert oracle.is_uniform(A[case["x"]]) == case["want"]


# -------------------------------------------------------------------- GPU


def _dev(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _code(a):
    from paper_2307_05389_b200.dtypes import CODE

    return CODE[np.dtype(a.dtype)]


@pytest.mark.gpu
def test_c_abi_width_and_uniform_ops(gold):
    import torch

    from paper_2307_05389_b200 import _lib

    L = _lib.load()
    ctx = _lib.context(0)
    c, A = gold
    for case in c["width"]:
        x = A[case["x"]]
        out = _dev(np.full(case["n_bins"] + 1, -7, np.int64))
        xd = _dev(x)
        rc = L.tsds_op_fill_width_offsets(ctx.handle, xd.data_ptr(), _code(x), x.shape[0], case["x0"], case["span"],
                                          case["n_bins"], case["k0"], case["k1"], out.data_ptr())
        _lib.check(rc, "fill_width_offsets")
        ctx.synchronize()
        assert np.array_equal(out.cpu().numpy(), A[case["want"]]), case
    for case in c["uniform"]:
        x = A[case["x"]]
        flag = torch.full((1,), -1, dtype=torch.int32, device="cuda")
        rc = L.tsds_op_is_uniform_spaced(ctx.handle, _dev(x).data_ptr(), _code(x), x.shape[0], flag.data_ptr())
        _lib.check(rc, "is_uniform_spaced")
        ctx.synchronize()
        assert bool(flag.item()) == case["want"], case


@pytest.mark.gpu
def test_c_abi_bin_writers_and_compaction(gold):
    import torch

    from paper_2307_05389_b200 import _lib

    L = _lib.load()
    ctx = _lib.context(0)
    c, A = gold
    for case in c["bins"]:
        y, off, w = A[case["y"]], A[case["off"]], case["width"]
        nb = off.shape[0] - 1
        idx = _dev(np.full(w * nb, -5, np.int64))
        cnt = _dev(np.full(nb, -5, np.int64))
        fn = L.tsds_op_minmax_bins if w == 2 else L.tsds_op_m4_bins
        yd, od = _dev(y), _dev(off)
        rc = fn(ctx.handle, yd.data_ptr(), _code(y), od.data_ptr(), case["b0"], case["b1"], 0, idx.data_ptr(),
                cnt.data_ptr())
        _lib.check(rc, "bins")
        ctx.synchronize()
        assert np.array_equal(idx.cpu().numpy(), A[case["idx"]]), (y.dtype, w, case["b0"], case["b1"])
        assert np.array_equal(cnt.cpu().numpy(), A[case["cnt"]]), (y.dtype, w, case["b0"], case["b1"])
    for case in c["compact"]:
        idx, cnt = _dev(A[case["idx"]]), _dev(A[case["cnt"]])
        out = torch.zeros(idx.numel() + 1, dtype=torch.int64, device="cuda")
        total = torch.zeros(1, dtype=torch.int64, device="cuda")
        rc = L.tsds_op_compact_bins(ctx.handle, idx.data_ptr(), cnt.data_ptr(), case["width"], cnt.numel(),
                                    out.data_ptr(), total.data_ptr())
        _lib.check(rc, "compact_bins")
        ctx.synchronize()
        want = A[case["want"]]
        assert int(total.item()) == want.shape[0]
        assert np.array_equal(out[: want.shape[0]].cpu().numpy(), want)


@pytest.mark.gpu
def test_c_abi_bin_writers_large_vs_oracle(oracle):
    """The writers over many bins and every dtype, NaN-propagating too."""
    import workloads as W
    from paper_2307_05389_b200 import _lib

    L = _lib.load()
    ctx = _lib.context(0)
    rng = np.random.default_rng(31)
    for tag in W.ALL_TAGS:
        y = W.random_series(tag, 400_003, int(rng.integers(1 << 30)), ties=True)
        if tag in ("f16", "f32", "f64"):
            y[rng.integers(0, y.shape[0], 500)] = np.nan
        nb = 3000
        off = np.sort(rng.integers(0, y.shape[0] + 1, nb + 1)).astype(np.int64)
        off[0], off[-1] = 0, y.shape[0]
        for w, nan in ((2, 0), (4, 0), (2, 1)):
            if nan and tag not in ("f16", "f32", "f64"):
                continue
            idx = _dev(np.full(w * nb, -5, np.int64))
            cnt = _dev(np.full(nb, -5, np.int64))
            fn = L.tsds_op_minmax_bins if w == 2 else L.tsds_op_m4_bins
            yd, od = _dev(y), _dev(off)
            _lib.check(fn(ctx.handle, yd.data_ptr(), _code(y), od.data_ptr(), 100, 2900, nan, idx.data_ptr(),
                          cnt.data_ptr()), "bins")
            ctx.synchronize()
            widx = np.full(w * nb, -5, np.int64)
            wcnt = np.full(nb, -5, np.int64)
            oracle.bins_slots(w, y, off, 100, 2900, widx, wcnt, nan=bool(nan))
            assert np.array_equal(cnt.cpu().numpy(), wcnt), (tag, w, nan)
            assert np.array_equal(idx.cpu().numpy(), widx), (tag, w, nan)


@pytest.mark.gpu
def test_c_abi_lttb_walk(gold):
    import torch

    from paper_2307_05389_b200 import _lib

    L = _lib.load()
    ctx = _lib.context(0)
    c, A = gold
    for case in c["lttb"]:
        y, off = A[case["y"]], A[case["off"]]
        nb = off.shape[0] - 1
        xf = None if case["x"] is None else _dev(A[case["x"]].astype(np.float64))
        out = torch.full((nb + 2,), -3, dtype=torch.int64, device="cuda")
        m = ctypes.c_int64(0)
        yd, od = _dev(y), _dev(off)
        rc = L.tsds_op_lttb(ctx.handle, None if xf is None else xf.data_ptr(), yd.data_ptr(), _code(y), y.shape[0],
                            od.data_ptr(), nb, out.data_ptr(), ctypes.byref(m))
        _lib.check(rc, "lttb")
        want = A[case["want"]]
        assert m.value == want.shape[0]
        assert np.array_equal(out[: want.shape[0]].cpu().numpy(), want), (y.dtype, case["x"] is None)


@pytest.mark.gpu
def test_estimator_transform_values(gold):
    import paper_2307_05389_b200 as ts

    c, A = gold
    for case in c["transform"]:
        est = getattr(ts, case["cls"])(**case["kw"])
        y = A[case["y"]]
        got_t = est.transform(y)
        got_ft = est.fit_transform(y)
        for got, key in ((got_t, "transform"), (got_ft, "fit_transform")):
            want = A[case[key]]
            assert got.dtype == want.dtype and got.shape == want.shape, (case["cls"], key)
            assert np.array_equal(got.view(np.uint8), want.view(np.uint8)), (case["cls"], key)
        # device input: values come back as a device tensor
        if y.dtype.kind != "u" or y.dtype.itemsize == 1:
            import torch

            got_d = est.transform(torch.from_numpy(y).cuda())
            assert np.array_equal(got_d.cpu().numpy().view(np.uint8), A[case["transform"]].view(np.uint8))


@pytest.mark.gpu
def test_cli_endpoint_bytes_match_reference(gold):
    """Same stdin bytes -> same stdout bytes and exit code as the reference CLI."""
    c, A = gold
    for case in c["cli"]:
        p = subprocess.run([sys.executable, "-m", "paper_2307_05389_b200", "downsample", *case["args"]],
                           input=A[case["stdin"]].tobytes(), capture_output=True, timeout=600,
                           cwd=os.path.dirname(HERE))
        assert p.returncode == case["code"], (case["args"], p.stderr.decode())
        assert p.stdout == A[case["stdout"]].tobytes(), case["args"]
        if case["code"] == 1:
            assert p.stderr.decode().strip().splitlines()[-1:] == case["stderr"], case["args"]
