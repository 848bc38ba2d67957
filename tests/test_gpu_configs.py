"""Full-size BASELINE configs C4 and C5 against the reference's outputs.

C4: MinMaxLTTB over 1e9 points (f64 x, f32 y, n_out 5000, ratio 4) equals
the reference's indices (tests/golden/configs.npz "c4_minmaxlttb", from
algorithms.py:211-255 run on the same seeded series), through host numpy
and through device tensors.  C5: every one of the 3 x 4096 series (i16,
f16, u8; 2e6 points, n_out 1000) matches the reference's per-series index
hash and count -- a checksum of checksums over 24.6e9 input bytes.
The inputs are regenerated with the process-parallel generators of
workloads.py (bit-identical to the sequential ones).
"""

import hashlib

import numpy as np
import pytest

import golden_io as G
import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ts():
    import paper_2307_05389_b200 as m

    return m


def _row_hash(row):
    return int.from_bytes(hashlib.blake2b(np.ascontiguousarray(row, dtype="<u8").tobytes(), digest_size=8).digest(),
                          "little")


def test_c4_config_full(ts):
    import torch

    g = G.configs()
    want = g["c4_minmaxlttb"]
    x, y = W.config4_parallel()
    got = ts.downsample("minmaxlttb", x, y, n_out=5000, minmax_ratio=4)
    assert got.dtype == np.uint64
    assert np.array_equal(got, want)
    est = ts.MinMaxLTTBDownsampler(n_out=5000, minmax_ratio=4)
    xd = torch.from_numpy(x).cuda()
    yd = torch.from_numpy(y).cuda()
    del x, y
    assert np.array_equal(est.downsample(xd, yd), want)
    # without x (positions stand in) the device path agrees with itself on a slice
    assert np.array_equal(ts.downsample("minmaxlttb", yd[:100_000_000], n_out=5000),
                          ts.downsample("minmaxlttb", yd[:100_000_000].cpu().numpy(), n_out=5000))


@pytest.mark.parametrize("tag", ["i16", "f16", "u8"])
def test_c5_all_series(ts, tag):
    g = G.configs()
    Y = W.config5_parallel(tag)
    idx, cnt = ts.minmax_batched(Y, n_out=1000)
    assert np.array_equal(cnt, g[f"c5_{tag}_count"])
    hashes = np.array([_row_hash(idx[s, : cnt[s]]) for s in range(Y.shape[0])], np.uint64)
    bad = np.nonzero(hashes != g[f"c5_{tag}_hash"])[0]
    assert bad.size == 0, (tag, bad[:10])
    for s in range(4):
        assert np.array_equal(idx[s, : cnt[s]], g[f"c5_{tag}_row{s}"])


def test_c5_device_batch_equals_host(ts):
    import torch

    Y = W.config5_parallel("i16", S=512)
    idx_h, cnt_h = ts.minmax_batched(Y, n_out=1000)
    idx_d, cnt_d = ts.minmax_batched(torch.from_numpy(Y).cuda(), n_out=1000)
    assert np.array_equal(cnt_h, cnt_d) and np.array_equal(idx_h, idx_d)


def test_uniform_device_x_is_dropped_for_minmaxlttb(ts, oracle):
    """Uniform x on the device: the reference drops it at the API
    level (api.py:19-28), so stage 2 bins the candidate positions by count."""
    import torch

    n = 20_000
    y = W.random_series("f64", n, 77)
    for x in (np.arange(n, dtype=np.int64) * 3 + 7, np.arange(n, dtype=np.float64) * 0.25):
        want = oracle.downsample("minmaxlttb", y, n_out=200, minmax_ratio=4)  # x dropped
        assert np.array_equal(ts.downsample("minmaxlttb", x, y, n_out=200, minmax_ratio=4), want)
        got = ts.downsample("minmaxlttb", torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), n_out=200,
                            minmax_ratio=4)
        assert np.array_equal(got, want)


def test_stale_status_is_not_reported(ts):
    """A device-x call that fails with "invalid index span" must not leak its
    status into later valid calls on the same context."""
    import torch

    from paper_2307_05389_b200 import _lib

    L = _lib.load()
    ctx = _lib.context(0)
    y = torch.from_numpy(W.random_series("f32", 10_000, 3)).cuda()
    xbad = torch.from_numpy(np.r_[np.zeros(9_999), [np.inf]]).cuda()
    out = torch.zeros(100, dtype=torch.int64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    rc = L.tsds_downsample_async(ctx.handle, 1, xbad.data_ptr(), 2, y.data_ptr(), 1, 10_000, 100, 4, 0, out.data_ptr(),
                                 cnt.data_ptr(), st.data_ptr())
    assert rc == 0
    ctx.synchronize()
    assert int(st.item()) == -2
    yh = y.cpu().numpy()
    # later valid calls without device binning
    assert ts.downsample("minmax", yh, n_out=100).shape[0] > 0
    assert ts.downsample("lttb", yh, n_out=100).shape[0] == 100
    rc = L.tsds_downsample_async(ctx.handle, 1, None, 0, y.data_ptr(), 1, 10_000, 100, 4, 0, out.data_ptr(),
                                 cnt.data_ptr(), st.data_ptr())
    assert rc == 0
    ctx.synchronize()
    assert int(st.item()) == 0


def test_calls_restore_callers_current_device(ts):
    import torch

    torch.cuda.set_device(0)
    y = W.random_series("f32", 50_000, 5)
    ts.downsample("minmax", y, n_out=100)
    assert torch.cuda.current_device() == 0


def test_async_api_all_algorithms_equal_sync(ts, oracle):
    """tsds_downsample_async (device pointers, no host round trip) for every
    algorithm, including MinMaxLTTB's on-device stage 2 with and without x,
    uniform x, m <= n_out (candidates returned) and a large ratio (host-sized
    stage 2), against the oracle."""
    import torch

    from paper_2307_05389_b200 import _lib

    L = _lib.load()
    ctx = _lib.context(0)
    rng = np.random.default_rng(5)
    n = 300_000
    y = np.cumsum(rng.standard_normal(n)).astype(np.float32)
    xs = {
        "none": None,
        "exp": np.cumsum(rng.exponential(1.0, n)),
        "gaps": np.cumsum(rng.integers(1, 4, n) * np.where(rng.random(n) < 0.001, 5000, 1)).astype(np.int64),
        "uniform": np.arange(n, dtype=np.int64) * 5 + 3,
    }
    yd = torch.from_numpy(y).cuda()
    algos = [("minmax", 1, 2000, 4), ("m4", 2, 2000, 4), ("lttb", 3, 1000, 4), ("minmaxlttb", 4, 1000, 4),
             ("minmaxlttb", 4, 500, 60), ("minmaxlttb", 4, 5000, 40), ("minmaxlttb", 4, 200, 1)]
    for xname, x in xs.items():
        xd = None if x is None else torch.from_numpy(x).cuda()
        for algo, code, n_out, ratio in algos:
            out = torch.full((n_out,), -1, dtype=torch.int64, device="cuda")
            cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
            st = torch.full((1,), 7, dtype=torch.int32, device="cuda")
            rc = L.tsds_downsample_async(ctx.handle, code, None if xd is None else xd.data_ptr(),
                                         0 if x is None else (2 if x.dtype == np.float64 else 6), yd.data_ptr(), 1, n,
                                         n_out, ratio, 0, out.data_ptr(), cnt.data_ptr(), st.data_ptr())
            _lib.check(rc, algo)
            ctx.synchronize()
            args = (y,) if x is None else (x, y)
            want = oracle.downsample(algo, *args, n_out=n_out, minmax_ratio=ratio)
            assert int(st.item()) == 0
            m = int(cnt.item())
            assert np.array_equal(out[:m].cpu().numpy(), want.astype(np.int64)), (xname, algo, n_out, ratio)


def test_lttb_device_x_invalid_span_raises(ts):
    import torch

    y = torch.from_numpy(W.random_series("f64", 50_000, 8)).cuda()
    x = np.cumsum(np.ones(50_000))
    x[-2] = np.inf  # interior slice x[1:-1] ends at +inf
    with pytest.raises(ValueError, match="invalid index span"):
        ts.downsample("lttb", torch.from_numpy(x).cuda(), y, n_out=500)
    with pytest.raises(ValueError, match="invalid index span"):
        ts.downsample("minmaxlttb", torch.from_numpy(x).cuda(), y, n_out=500)
    # the context stays usable
    assert ts.downsample("lttb", y, n_out=500).shape[0] == 500
