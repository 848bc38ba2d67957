"""Pin-on-reuse cache of large host inputs (paper_2307_05389_b200/pinning.py)."""

import gc

import numpy as np
import pytest

from paper_2307_05389_b200 import pinning


def test_owner_resolution():
    a = np.arange(1000, dtype=np.float32)
    assert pinning.owner_of(a) is a
    assert pinning.owner_of(a[10:500]) is a
    assert pinning.owner_of(a[10:500].view(np.int32)[::1]) is a
    b = np.frombuffer(bytearray(64), dtype=np.uint8)  # a buffer export keeps the memory alive while b lives
    assert pinning.owner_of(b) is b and pinning.owner_of(b[8:].view(np.int16)) is b
    import mmap

    m = np.frombuffer(mmap.mmap(-1, 4096), dtype=np.float32).reshape(32, 32)
    assert pinning.owner_of(m[3:]) is m.base

    class Foreign:  # memory whose lifetime numpy cannot vouch for
        __array_interface__ = a.__array_interface__

    assert pinning.owner_of(np.asarray(Foreign())) is None


def test_small_or_disabled_inputs_are_ignored():
    a = np.zeros(1000, dtype=np.float64)
    assert pinning.note_host_input(a) is False  # below the threshold: no library call at all
    assert pinning.pinned_bytes() == 0


@pytest.mark.gpu
def test_pin_on_second_call_and_release_on_collect():
    import paper_2307_05389_b200 as ts
    from oracle import oracle as O

    pinning.release_all()
    pinning.configure(mode="reuse", min_bytes=1 << 20)
    try:
        rng = np.random.default_rng(3)
        y = np.cumsum(rng.standard_normal(3_000_000)).astype(np.float32)  # 12 MB
        want = O.downsample("minmax", y, n_out=2000)
        reg0, rel0 = pinning.stats["registered"], pinning.stats["released"]
        assert np.array_equal(ts.downsample("minmax", y, n_out=2000), want)
        assert pinning.pinned_bytes() == 0  # first sight: staged
        assert np.array_equal(ts.downsample("minmax", y, n_out=2000), want)
        assert pinning.pinned_bytes() == y.nbytes and pinning.stats["registered"] == reg0 + 1
        # a view of the same buffer reuses the registration
        assert np.array_equal(ts.downsample("m4", y[1000:], n_out=400), O.downsample("m4", y[1000:], n_out=400))
        assert pinning.stats["registered"] == reg0 + 1
        del y
        gc.collect()
        assert pinning.pinned_bytes() == 0 and pinning.stats["released"] == rel0 + 1
    finally:
        pinning.configure(mode="reuse", min_bytes=64 << 20)
        pinning.release_all()
