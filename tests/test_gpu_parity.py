"""GPU parity: the CUDA path (through libtsds.so) against the reference.

Expected values come from the golden fixtures made by importing the real
reference (tests/golden/make_golden.py), or from the pinned CPU oracle at
sizes where no fixture exists.  Index work is bit-exact: every comparison
is array equality.
"""

import numpy as np
import pytest

import golden_io as G
import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ts():
    import paper_2307_05389_b200 as m

    return m


def _args(x, y):
    return (y,) if x is None else (x, y)


@pytest.mark.parametrize("algo", ["minmax", "m4", "lttb", "minmaxlttb"])
def test_sweep_matches_reference(ts, algo):
    n = 0
    for rec, x, y, want, _ in G.sweep(algo):
        kw = {"minmax_ratio": rec["ratio"]} if algo == "minmaxlttb" else {}
        got = ts.downsample(algo, *_args(x, y), n_out=rec["n_out"], **kw)
        assert got.dtype == np.uint64
        assert got.tolist() == want.tolist(), rec
        n += 1
    assert n >= 80


def test_argminmax_cases(ts):
    c, A = G.cases()
    for case in c["argminmax"]:
        assert list(ts.argminmax(A[case["y"]])) == case["want"], case["note"]


def test_downsample_cases(ts):
    c, A = G.cases()
    for case in c["downsample"]:
        y = A[case["y"]]
        args = (y,) if case["x"] is None else (A[case["x"]], y)
        got = ts.downsample(case["algo"], *args, n_out=case["n_out"], **case["kw"])
        assert got.tolist() == case["want"], (case["algo"], case["note"])


def test_equal_width_cases_host_and_device(ts):
    import torch

    c, A = G.cases()
    for case in c["equal_width"]:
        x = A[case["x"]]
        if case["error"]:
            with pytest.raises(ValueError, match=case["error"]):
                ts.equal_width_boundaries(x, case["n_bins"])
            continue
        assert ts.equal_width_boundaries(x, case["n_bins"]).tolist() == case["want"], case["note"]
        if x.shape[0] and x.dtype != np.uint32 and x.dtype != np.uint64:
            xd = torch.from_numpy(x).cuda()
            assert ts.equal_width_boundaries(xd, case["n_bins"]).tolist() == case["want"], case["note"]


@pytest.mark.parametrize("algo", ["minmax", "m4", "minmaxlttb"])
def test_nan_propagating_vs_oracle(ts, oracle, algo):
    for i, tag in enumerate(["f16", "f32", "f64"] * 4):
        n = [777, 5000, 20_000, 100_003][i // 3]
        y = W.nan_series(tag, n, 40 + i, frac=0.002, at_starts=[0, n // 3])
        n_out = 64 if algo != "minmaxlttb" else 50
        got = ts.downsample("nan" + algo, y, n_out=n_out)
        want = oracle.downsample(algo, y, n_out=n_out, nan=True)
        assert got.tolist() == want.tolist(), (algo, tag, n)
        plain = ts.downsample(algo, y, n_out=n_out)
        assert plain.tolist() == oracle.downsample(algo, y, n_out=n_out).tolist(), (algo, tag, n)


def test_device_inputs_equal_host(ts):
    import torch

    for rec, x, y, want, _ in list(G.sweep("m4"))[:30]:
        if y.dtype in (np.uint16, np.uint32, np.uint64) or (x is not None and x.dtype in (np.uint32, np.uint64)):
            continue
        yd = torch.from_numpy(y).cuda()
        xd = None if x is None else torch.from_numpy(x).cuda()
        got = ts.downsample("m4", *_args(xd, yd), n_out=rec["n_out"])
        assert got.tolist() == want.tolist(), rec
    for rec, x, y, want, _ in list(G.sweep("minmaxlttb"))[:30]:
        if y.dtype in (np.uint16, np.uint32, np.uint64) or (x is not None and x.dtype in (np.uint32, np.uint64)):
            continue
        yd = torch.from_numpy(y).cuda()
        xd = None if x is None else torch.from_numpy(x).cuda()
        got = ts.downsample("minmaxlttb", *_args(xd, yd), n_out=rec["n_out"], minmax_ratio=rec["ratio"])
        assert got.tolist() == want.tolist(), rec


def test_misaligned_and_tiny_bins(ts, oracle):
    # slices that start at every offset within a 16-byte vector, bins of 1..70 elements
    base = W.random_series("f32", 50_000, 3, ties=True)
    for off in range(0, 5):
        y = base[off:]
        for n_out in (2, 4, 10, 1000, 20_000, 49_990):
            got = ts.downsample("minmax", y, n_out=n_out)
            assert got.tolist() == oracle.downsample("minmax", y, n_out=n_out).tolist(), (off, n_out)
    for tag in W.ALL_TAGS:
        y = W.random_series(tag, 30_001, 9, ties=True)[1:]
        for n_out in (4, 8, 400, 7_500):
            got = ts.downsample("m4", y, n_out=n_out)
            assert got.tolist() == oracle.downsample("m4", y, n_out=n_out).tolist(), (tag, n_out)


def test_all_equal_and_extreme_values(ts, oracle):
    for tag in W.ALL_TAGS:
        dt = W.DTYPES[tag]
        for fill in ("zero", "max", "min"):
            if fill == "zero":
                y = np.zeros(70_001, dt)
            elif dt in (np.float16, np.float32, np.float64):
                y = np.full(70_001, np.inf if fill == "max" else -np.inf, dt)
            else:
                info = np.iinfo(dt)
                y = np.full(70_001, info.max if fill == "max" else info.min, dt)
            for algo, n_out in (("minmax", 40), ("m4", 40), ("minmaxlttb", 30)):
                got = ts.downsample(algo, y, n_out=n_out)
                assert got.tolist() == oracle.downsample(algo, y, n_out=n_out).tolist(), (tag, fill, algo)


def test_whole_array_argminmax_large(ts, oracle):
    for tag in ("f32", "u8", "i64", "f16"):
        y = W.random_series(tag, 5_000_017, 5, ties=True)
        assert ts.argminmax(y) == oracle.argminmax(y), tag


def test_batched_rows_equal_single(ts, oracle):
    for tag in ("i16", "u8", "f16"):
        Y = W.config5(tag, S=24, L=200_000)
        idx, cnt = ts.minmax_batched(Y, n_out=1000)
        want, wcnt = oracle.minmax_batched(Y, n_out=1000)
        assert np.array_equal(cnt, wcnt)
        for s in range(Y.shape[0]):
            assert idx[s, : cnt[s]].tolist() == want[s, : wcnt[s]].tolist(), (tag, s)


def test_batched_thread_per_bin_kernel(ts, oracle):
    """The lane-group batched kernel (8 lanes per bin; forced on for small inputs): every
    width, ties, f16 +-0/NaN ordering, f32 NaNs, and bins that do not start
    or end on a 16-byte boundary (head/tail elements)."""
    from paper_2307_05389_b200 import _lib

    L = _lib.load()
    rng = np.random.default_rng(12)
    try:
        L.tsds_set_option(b"lane_bins", 2)
        for tag in ("u8", "i8", "i16", "u16", "f16", "f32", "i32", "u64", "f64"):
            for length, n_out in ((20_000, 100), (20_011, 98), (4_003, 1000)):
                Y = np.stack([W.random_series(tag, length, int(rng.integers(1 << 30)), ties=True) for _ in range(5)])
                if tag in ("f32", "f64"):
                    Y[1, ::97] = np.nan
                    Y[2, :] = np.nan
                if tag == "f16":
                    Y[1, ::53] = -0.0
                    Y[1, 7::61] = 0.0
                    Y[2, ::71] = np.float16("nan")
                    Y[3].view(np.uint16)[5::89] = 0xFE00  # negative NaN pattern (ordinal: below -inf)
                    Y[4, ::37] = -np.inf
                idx, cnt = ts.minmax_batched(Y, n_out=n_out)
                want, wcnt = oracle.minmax_batched(Y, n_out=n_out)
                assert np.array_equal(cnt, wcnt), (tag, length)
                for s in range(Y.shape[0]):
                    assert idx[s, : cnt[s]].tolist() == want[s, : wcnt[s]].tolist(), (tag, length, s)
    finally:
        L.tsds_set_option(b"lane_bins", 1)


def test_cta_per_bin_scan_mode(ts, oracle):
    """Small inputs with >= #SM bins take the CTA-per-bin scan (C1's path):
    MinMax / M4 / NaN-propagating, with and without x, every width."""
    rng = np.random.default_rng(21)
    for tag in ("f32", "f64", "f16", "i64", "u8", "i16", "u32"):
        y = W.random_series(tag, 300_001, int(rng.integers(1 << 30)), ties=True)
        if tag in ("f32", "f64"):
            y[rng.integers(0, y.size, 300)] = np.nan
        x = np.cumsum(rng.integers(1, 9, y.size)).astype(np.int64)
        for algo in ("minmax", "m4"):
            assert ts.downsample(algo, y, n_out=2000).tolist() == oracle.downsample(algo, y, n_out=2000).tolist(), (tag, algo)
            assert ts.downsample(algo, x, y, n_out=2000).tolist() == oracle.downsample(algo, x, y, n_out=2000).tolist(), (tag, algo, "x")
        if tag in ("f32", "f64", "f16"):
            got = ts.downsample("nanm4", y, n_out=2000).tolist()
            assert got == oracle.downsample("m4", y, n_out=2000, nan=True).tolist(), (tag, "nanm4")


def test_c1_config(ts):
    g = G.configs()
    y = W.config1()
    assert ts.downsample("minmax", y, n_out=2000).tolist() == g["c1_minmax"].tolist()


def test_c2_config_m4_and_nanm4(ts, oracle):
    import torch

    g = G.configs()
    x, y = W.config2()
    assert ts.downsample("m4", x, y, n_out=4000).tolist() == g["c2_m4"].tolist()
    assert ts.downsample("minmax", x, y, n_out=4000).tolist() == g["c2_minmax"].tolist()
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    assert ts.downsample("m4", xd, yd, n_out=4000).tolist() == g["c2_m4"].tolist()
    want_nan = oracle.downsample("m4", x, y, n_out=4000, nan=True, threads=8)
    assert ts.downsample("nanm4", xd, yd, n_out=4000).tolist() == want_nan.tolist()


def test_c3_config_lttb(ts):
    """C3 against the reference; a differing pick is only allowed inside a
    bucket whose two best areas are within 1e-12 (counted and printed)."""
    from lttb_ties import explain_mismatches, lttb_offsets

    g = G.configs()
    y = W.config3()
    for n_out in (1000, 10000):
        got = ts.downsample("lttb", y, n_out=n_out)
        want = g[f"c3_lttb_{n_out}"]
        mism = explain_mismatches(got, want, y, lttb_offsets(y.shape[0], n_out))
        print(f"C3 n_out={n_out}: picks differing at near-ties = {mism}")


def test_c5_first_series_hashes(ts):
    import hashlib

    g = G.configs()
    for tag in ("i16", "f16", "u8"):
        Y = W.config5(tag, S=16)
        idx, cnt = ts.minmax_batched(Y, n_out=1000)
        for s in range(16):
            row = idx[s, : cnt[s]]
            h = int.from_bytes(hashlib.blake2b(row.astype("<u8").tobytes(), digest_size=8).digest(), "little")
            assert h == int(g[f"c5_{tag}_hash"][s]), (tag, s)


def test_lttb_large_bucket_modes(ts, oracle):
    """Guess/verify LTTB with the reference's sequential centroids (exact=1)
    is bit-exact; tree-summed centroids (exact=2) match here too (SURVEY
    probe 8 found no near-ties on such data)."""
    from paper_2307_05389_b200 import _lib

    L = _lib.load()
    y = W.config3(2_000_000)
    x = np.cumsum(np.random.default_rng(4).exponential(1.0, y.shape[0]))
    try:
        for mode in (1, 2, 0):
            L.tsds_set_option(b"lttb_exact", mode)
            for n_out in (50, 1000):
                assert ts.downsample("lttb", y, n_out=n_out).tolist() == oracle.downsample("lttb", y, n_out=n_out).tolist()
                assert ts.downsample("lttb", x, y, n_out=n_out).tolist() == oracle.downsample("lttb", x, y, n_out=n_out).tolist()
            steps = L.tsds_ctx_stat(_lib.context().handle, b"lttb_rounds")  # correction-chain steps
            assert 0 <= steps <= 4 * 1000
    finally:
        L.tsds_set_option(b"lttb_exact", 0)


@pytest.mark.gpu
def test_lttb_large_vector_paths(ts, oracle):
    """Large-bucket LTTB through the 128-bit vector paths for every value
    width, with exact ties (u8), NaNs, many buckets (multi-block layout scan)
    and a misaligned device input (scalar fallback)."""
    import torch

    rng = np.random.default_rng(11)
    base = np.cumsum(rng.laplace(size=600_000))
    withnan = base.copy()
    withnan[rng.integers(0, base.size, 64)] = np.nan
    cases = [
        base,
        withnan,
        base.astype(np.float32),
        base.astype(np.float16),
        (base * 50).astype(np.int64),
        np.clip(base * 3, -32768, 32767).astype(np.int16),
        (np.abs(base) % 250).astype(np.uint8),
        (np.abs(base) * 7).astype(np.uint32),
    ]
    withinf = base.copy()
    withinf[rng.integers(0, base.size, 8)] = np.inf
    withinf[rng.integers(0, base.size, 8)] = -np.inf
    cases += [withinf, np.full(200_000, 3.25), np.full(200_000, np.nan)]
    for y in cases:
        for n_out in (300, 15_000):  # avg bucket 2000 and 40: both on the large path
            got = ts.downsample("lttb", y, n_out=n_out)
            assert got.tolist() == oracle.downsample("lttb", y, n_out=n_out).tolist(), (y.dtype, n_out)
    big = np.cumsum(rng.laplace(size=2_500_000))
    assert ts.downsample("lttb", big, n_out=60_000).tolist() == oracle.downsample("lttb", big, n_out=60_000).tolist()
    yd = torch.from_numpy(base).cuda()[1:]
    assert ts.downsample("lttb", yd, n_out=1000).tolist() == oracle.downsample("lttb", base[1:], n_out=1000).tolist()


@pytest.mark.parametrize("mode", [0, 2])
def test_atomic_bin_merge_mode(ts, oracle, mode):
    """Atomic merge mode (64-bit packed (key, index) atomics + dependent
    compaction kernel) forced on (2) and off (0): every <= 32-bit dtype,
    ties, NaN in first slots, NaN-propagating, device x with non-monotone
    offsets, the slot writers and MinMaxLTTB preselection."""
    import torch

    from paper_2307_05389_b200 import _lib

    L = _lib.load()
    rng = np.random.default_rng(41)
    try:
        L.tsds_set_option(b"atomic_bins", mode)
        for tag in ("f32", "f16", "i8", "u8", "i16", "u16", "i32", "u32"):
            y = W.random_series(tag, 250_003, int(rng.integers(1 << 30)), ties=True)
            if tag in ("f32", "f16"):
                y[rng.integers(0, y.size, 200)] = np.nan
                y[[0, 1250, 2500]] = np.nan
            x = np.cumsum(rng.integers(1, 9, y.size)).astype(np.int64)
            for algo, n_out in (("minmax", 2000), ("m4", 400), ("minmax", 6), ("minmaxlttb", 300)):
                want = oracle.downsample(algo, y, n_out=n_out)
                assert ts.downsample(algo, y, n_out=n_out).tolist() == want.tolist(), (tag, algo, n_out)
                want = oracle.downsample(algo, x, y, n_out=n_out)
                assert ts.downsample(algo, torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(),
                                     n_out=n_out).tolist() == want.tolist(), (tag, algo, n_out, "dev x")
            if tag in ("f32", "f16"):
                got = ts.downsample("nanm4", y, n_out=2000).tolist()
                assert got == oracle.downsample("m4", y, n_out=2000, nan=True).tolist(), (tag, "nanm4")
        # non-monotone device x: independent bins
        y = W.random_series("f32", 100_000, 3, ties=True)
        x = np.cumsum(rng.integers(1, 9, y.size)).astype(np.int64)
        x[50_000:50_100] = x[50_000:50_100][::-1]
        want = oracle.downsample("minmax", x, y, n_out=1000)
        assert ts.downsample("minmax", torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(),
                             n_out=1000).tolist() == want.tolist()
    finally:
        L.tsds_set_option(b"atomic_bins", 1)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [2, 0])
def test_tile_bins_kernel(ts, oracle, mode):
    """Bins streamed through shared memory by TMA bulk copies (C1's path),
    forced on for every shape (2) and off (0): every dtype, ties, NaN in a
    bin's first slot, NaN-propagating, host x (offset arrays, empty bins),
    bins longer than a slot (tile by tile), tiny bins, misaligned starts,
    MinMaxLTTB preselection; the direct output layout and its fallback."""
    import torch

    from paper_2307_05389_b200 import _lib

    L = _lib.load()
    rng = np.random.default_rng(77)
    try:
        L.tsds_set_option(b"tile_bins", mode)
        for tag in ("f32", "f64", "f16", "i8", "u8", "i16", "u16", "i32", "u32", "i64", "u64"):
            y = W.random_series(tag, 250_003, int(rng.integers(1 << 30)), ties=True)
            if tag in ("f32", "f64", "f16"):
                y[rng.integers(0, y.size, 200)] = np.nan
                y[[0, 1250, 2500]] = np.nan
            x = np.cumsum(rng.integers(1, 9, y.size)).astype(np.int64)
            x[100_000:] += 40_000  # a gap: empty bins with many bins
            # ... ("minmax", 200_000): > 512 bins per CTA, i.e. several passes over the CTA's bin table
            for algo, n_out in (("minmax", 2000), ("m4", 400), ("minmax", 6), ("m4", 4), ("minmax", 50_000),
                                ("minmax", 200_000), ("minmaxlttb", 300)):
                want = oracle.downsample(algo, y, n_out=n_out)
                assert ts.downsample(algo, y, n_out=n_out).tolist() == want.tolist(), (tag, algo, n_out)
                want = oracle.downsample(algo, x, y, n_out=n_out)
                assert ts.downsample(algo, x, y, n_out=n_out).tolist() == want.tolist(), (tag, algo, n_out, "host x")
            yd = torch.from_numpy(y).cuda()
            for o in (1, 3):  # device views starting off a 16-byte boundary
                assert ts.downsample("m4", yd[o:], n_out=400).tolist() == oracle.downsample("m4", y[o:], n_out=400).tolist()
            if tag in ("f32", "f64", "f16"):
                got = ts.downsample("nanm4", y, n_out=2000).tolist()
                assert got == oracle.downsample("m4", y, n_out=2000, nan=True).tolist(), (tag, "nanm4")
        # constant series: every bin emits one index (the direct layout's fallback)
        c = np.full(100_000, 2.5, np.float32)
        assert ts.downsample("minmax", c, n_out=1000).tolist() == oracle.downsample("minmax", c, n_out=1000).tolist()
        assert ts.downsample("m4", c, n_out=1000).tolist() == oracle.downsample("m4", c, n_out=1000).tolist()
        # repeated calls: the flag reset between launches
        y = W.config1(1_000_000)
        want = oracle.downsample("minmax", y, n_out=2000).tolist()
        for _ in range(5):
            assert ts.downsample("minmax", y, n_out=2000).tolist() == want
    finally:
        L.tsds_set_option(b"tile_bins", 1)
