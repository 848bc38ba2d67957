"""Pin the CPU oracle (oracle/tsds_oracle.c) to the real reference.

Every expected value here was produced by importing the unmodified
reference (thinseries, forced scalar level) -- see tests/golden/make_golden.py.
"""

import hashlib

import numpy as np
import pytest

import golden_io as G


def _input_hash(x, y):
    h = hashlib.blake2b(digest_size=8)
    if x is not None:
        h.update(np.ascontiguousarray(x).tobytes())
    h.update(np.ascontiguousarray(y).tobytes())
    return int.from_bytes(h.digest(), "little")


@pytest.mark.parametrize("algo", ["minmax", "m4", "lttb", "minmaxlttb"])
def test_oracle_matches_reference_sweep(oracle, algo):
    n = 0
    for rec, x, y, want, ih in G.sweep(algo):
        assert _input_hash(x, y) == ih, ("workload generator drifted", rec)
        args = (y,) if x is None else (x, y)
        got = oracle.downsample(algo, *args, n_out=rec["n_out"], minmax_ratio=rec["ratio"])
        assert got.tolist() == want.tolist(), rec
        n += 1
    assert n >= 80


def test_oracle_argminmax_cases(oracle):
    c, A = G.cases()
    for case in c["argminmax"]:
        y = A[case["y"]]
        assert list(oracle.argminmax(y)) == case["want"], case["note"]


def test_oracle_binning_cases(oracle):
    c, A = G.cases()
    for case in c["equal_count"]:
        assert oracle.equal_count(case["length"], case["n_bins"]).tolist() == case["want"]
    for case in c["equal_width"]:
        x = A[case["x"]]
        if case["error"]:
            with pytest.raises(ValueError, match=case["error"]):
                oracle.equal_width(x, case["n_bins"])
        else:
            assert oracle.equal_width(x, case["n_bins"]).tolist() == case["want"], case["note"]


def test_oracle_downsample_cases(oracle):
    c, A = G.cases()
    for case in c["downsample"]:
        y = A[case["y"]]
        args = (y,) if case["x"] is None else (A[case["x"]], y)
        got = oracle.downsample(case["algo"], *args, n_out=case["n_out"], **case["kw"])
        assert got.tolist() == case["want"], (case["algo"], case["note"])


def test_oracle_threads_equal_sequential(oracle):
    import workloads as W

    y = W.random_series("f32", 200_000, 3, ties=True)
    for algo in ("minmax", "m4", "minmaxlttb"):
        a = oracle.downsample(algo, y, n_out=400, threads=1)
        b = oracle.downsample(algo, y, n_out=400, threads=7)
        assert np.array_equal(a, b)
