"""CPU-only checks of the product surface: the C ABI library loads and
exports every symbol include/tsds.h declares, validation errors match the
reference's exact strings (raised before any kernel runs), and the host-side
binning helpers equal the golden reference offsets."""

import os
import re

import numpy as np
import pytest

import golden_io as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    from paper_2307_05389_b200 import _lib

    with open(os.path.join(ROOT, "include", "tsds.h")) as f:
        hdr = f.read()
    declared = set(re.findall(r"\b(tsds_[a-z0-9_]+)\s*\(", hdr))
    assert len(declared) >= 20
    L = _lib.load()
    for name in sorted(declared):
        assert hasattr(L, name), name
    assert declared == set(_lib.EXPORTED)
    assert L.tsds_version() >= 100


def test_no_gpu_fails_loudly_not_silently():
    import paper_2307_05389_b200 as ts
    from paper_2307_05389_b200 import _lib

    if _lib.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError):
        ts.downsample("minmax", np.arange(100, dtype=np.float32), n_out=10)


def test_error_strings_match_reference():
    import paper_2307_05389_b200 as ts

    c, _ = G.cases()
    z = np.zeros(10, np.float64)
    calls = {
        "unknown algorithm": ("nope", (z,), {"n_out": 3}),
        "odd n_out": ("minmax", (z,), {"n_out": 5}),
        "empty": ("minmax", (np.array([], np.float64),), {"n_out": 4}),
        "n_out 0": ("minmax", (z,), {"n_out": 0}),
        "m4 n_out": ("m4", (z,), {"n_out": 6}),
        "lttb small": ("lttb", (z,), {"n_out": 2}),
        "ratio": ("minmaxlttb", (z,), {"n_out": 4, "minmax_ratio": 0}),
        "length mismatch": ("minmax", (np.arange(4), z[:5]), {"n_out": 4}),
        "unsupported dtype": ("minmax", (np.zeros(5, np.complex128),), {"n_out": 4}),
        "unknown kw": ("minmax", (z,), {"n_out": 4, "bogus": 1}),
        "kw on lttb": ("lttb", (z,), {"n_out": 4, "minmax_ratio": 2}),
        "bad workers": ("minmax", (z,), {"n_out": 4, "workers": 0}),
        "2-D": ("minmax", (np.zeros((2, 5)),), {"n_out": 4}),
        "non-contiguous": ("minmax", (np.zeros(20)[::2],), {"n_out": 4}),
        "f16 x": ("minmax", (np.zeros(5, np.float16), np.zeros(5)), {"n_out": 4}),
        "three args": ("minmax", (z, z, z), {"n_out": 4}),
    }
    checked = 0
    for case in c["errors"]:
        if case["note"] not in calls:
            continue
        algo, args, kw = calls[case["note"]]
        kind, msg = case["error"].split(": ", 1)
        with pytest.raises((ValueError, TypeError)) as ei:
            ts.downsample(algo, *args, **kw)
        assert type(ei.value).__name__ == kind, case["note"]
        assert str(ei.value) == msg, case["note"]
        checked += 1
    assert checked == len(calls)


def test_identity_and_everynth_need_no_gpu():
    import paper_2307_05389_b200 as ts

    y = np.arange(8, dtype=np.int64)
    for algo, n_out in (("minmax", 8), ("m4", 8), ("lttb", 8), ("minmaxlttb", 8)):
        got = ts.downsample(algo, y, n_out=n_out)
        assert got.dtype == np.uint64 and got.tolist() == list(range(8))
    assert ts.downsample("everynth", np.zeros(10, np.float32), n_out=5).tolist() == [0, 2, 4, 6, 8]
    assert ts.downsample("minmax", np.zeros(40), n_out=40, workers=0).tolist() == list(range(40))


def test_estimator_surface():
    import paper_2307_05389_b200 as ts

    est = ts.MinMaxLTTBDownsampler(n_out=128, parallel=True, minmax_ratio=2)
    assert est.get_params() == {"n_out": 128, "parallel": True, "minmax_ratio": 2}
    est.set_params(n_out=64, parallel=False)
    assert est.get_params()["n_out"] == 64
    with pytest.raises(ValueError, match="invalid parameter"):
        est.set_params(whatever=3)
    assert ts.NaNM4Downsampler().get_params() == {"n_out": 2000, "parallel": False}
    sklearn = pytest.importorskip("sklearn")
    from sklearn.base import clone

    dup = clone(ts.MinMaxLTTBDownsampler(n_out=77, minmax_ratio=3))
    assert dup.get_params()["minmax_ratio"] == 3


def test_host_binning_matches_reference_offsets():
    import paper_2307_05389_b200 as ts

    c, A = G.cases()
    for case in c["equal_count"]:
        assert ts.equal_count_boundaries(case["length"], case["n_bins"]).tolist() == case["want"]
    for case in c["equal_width"]:
        x = A[case["x"]]
        if case["error"]:
            with pytest.raises(ValueError, match=case["error"]):
                ts.equal_width_boundaries(x, case["n_bins"])
        else:
            assert ts.equal_width_boundaries(x, case["n_bins"]).tolist() == case["want"], case["note"]
    with pytest.raises(ValueError, match="invalid bin count"):
        ts.equal_count_boundaries(10, 0)
    with pytest.raises(ValueError, match="invalid worker count"):
        ts.boundaries_parallel(None, 10, 2, 0)


def test_ordinal_transforms_exhaustive():
    import paper_2307_05389_b200 as ts

    pats = np.arange(65536, dtype=np.uint16).view(np.int16)
    once = ts.ord_transform_i16(pats)
    assert np.array_equal(ts.ord_transform_i16(once), pats)
    want = np.array([(((0xFFFF if (p >> 15) & 1 else 0) & 0x7FFF) ^ p) & 0xFFFF for p in range(65536)], np.uint16)
    assert np.array_equal(once.view(np.uint16), want)
    u8 = np.arange(256, dtype=np.uint8)
    k = ts.ord_transform_uint(u8)
    assert k.dtype == np.int8 and np.all(np.diff(k.astype(np.int64)) > 0)
    assert np.array_equal(ts.ord_transform_uint(k), u8)
