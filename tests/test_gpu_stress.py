"""Repeat-and-compare stress over the kernels that synchronise across CTAs
(last-arriver merges, tickets, packed atomics, the TMA slot ring, LTTB
correction chains and locks).  compute-sanitizer is closed on the GPU pool
(tools/sanitize.sh records its refusal), so races are hunted the other way:
every protocol runs many times on changing inputs and launch geometries and
must return the oracle's answer every time -- a lost update or a stale
counter shows up as a differing index or a hang (pytest-timeout)."""

import threading

import numpy as np
import pytest

import workloads as W

pytestmark = pytest.mark.gpu


def _opts(L, **kw):
    for k, v in kw.items():
        L.tsds_set_option(k.encode(), v)


@pytest.mark.timeout(600)
def test_repeated_runs_every_merge_protocol(ts, oracle):
    import torch

    from paper_2307_05389_b200 import _lib

    L = _lib.load()
    rng = np.random.default_rng(2024)
    modes = [
        dict(tile_bins=0, atomic_bins=0),  # warp chunks: per-bin arrival counters, last-arriver merge, last-CTA ticket
        dict(tile_bins=0, atomic_bins=2),  # packed 64-bit atomics + dependent finish kernel
        dict(tile_bins=2, atomic_bins=0),  # TMA slot ring, named barriers, direct output + fallback flag
    ]
    try:
        for mode in modes:
            _opts(L, **mode)
            for rep in range(12):
                n = int(rng.integers(200_000, 900_000))
                tag = ("f32", "i16", "u8", "f64")[rep % 4]
                y = W.random_series(tag, n, int(rng.integers(1 << 30)), ties=True)
                yd = torch.from_numpy(y).cuda()
                for algo, n_out in (("minmax", 2000), ("m4", 8), ("m4", 4000), ("minmax", 40)):
                    if mode.get("atomic_bins") == 2 and tag == "f64":
                        continue
                    want = oracle.downsample(algo, y, n_out=n_out).tolist()
                    for _ in range(3):
                        assert ts.downsample(algo, yd, n_out=n_out).tolist() == want, (mode, tag, n, algo, n_out)
    finally:
        _opts(L, tile_bins=1, atomic_bins=1)


@pytest.mark.timeout(600)
def test_repeated_lttb_chains_and_batches(ts, oracle):
    import torch

    rng = np.random.default_rng(7)
    for rep in range(6):
        n = int(rng.integers(400_000, 1_500_000))
        y = np.cumsum(rng.laplace(size=n))
        y[rng.integers(0, n, 20)] += 50.0
        yd = torch.from_numpy(y).cuda()
        for n_out in (60, 1500, 9000):
            want = oracle.downsample("lttb", y, n_out=n_out).tolist()
            for _ in range(3):
                assert ts.downsample("lttb", yd, n_out=n_out).tolist() == want, (rep, n, n_out)
        want = oracle.downsample("minmaxlttb", y, n_out=500).tolist()
        for _ in range(3):
            assert ts.downsample("minmaxlttb", yd, n_out=500).tolist() == want
    for tag in ("u8", "f16", "i16"):
        Y = W.config5(tag, S=37, L=150_000)
        want, wcnt = oracle.minmax_batched(Y, n_out=1000)
        for _ in range(4):
            idx, cnt = ts.minmax_batched(Y, n_out=1000)
            assert np.array_equal(cnt, wcnt) and all(np.array_equal(idx[s, : cnt[s]], want[s, : wcnt[s]]) for s in range(37))


@pytest.mark.timeout(600)
def test_two_threads_two_contexts(ts, oracle):
    """Contexts are per thread: concurrent callers on one device must not disturb each other."""
    y1 = W.config1(3_000_000)
    x2, y2 = W.config2(2_000_000)
    want1 = oracle.downsample("minmax", y1, n_out=2000).tolist()
    want2 = oracle.downsample("m4", x2, y2, n_out=4000).tolist()
    bad = []

    def run(fn, want):
        for _ in range(15):
            if fn().tolist() != want:
                bad.append(1)

    t1 = threading.Thread(target=run, args=(lambda: ts.downsample("minmax", y1, n_out=2000), want1))
    t2 = threading.Thread(target=run, args=(lambda: ts.downsample("m4", x2, y2, n_out=4000), want2))
    t1.start(); t2.start(); t1.join(); t2.join()
    assert not bad
