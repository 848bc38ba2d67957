"""Bin boundaries (mirrors thinseries.binning, binning.py:1-138).

These public helpers return host numpy offsets like the reference.  Host x
is binned by libtsds's host binning (tsds_host_equal_width_offsets, exact
reference semantics); device x by the device kernels
(tsds_op_equal_width_offsets: uniform check + warp-cooperative exact binary
search).  `boundaries_parallel` exists for parity: the result never depends
on `workers` (as in the reference, binning.py:85-125).
"""

import numpy as np

from . import _lib
from .dtypes import CODE, as_index_series, is_device, length


def equal_count_boundaries(length_, n_bins):
    """offsets[k] = floor(k * length / n_bins) (binning.py:32-40)."""
    if n_bins < 1:
        raise ValueError("invalid bin count")
    k = np.arange(0, n_bins + 1, dtype=np.int64)
    return (k * np.int64(length_) // np.int64(n_bins)).astype(np.uint64)


def equal_width_boundaries(x, n_bins):
    """Equal x-width bins located by binary search (binning.py:61-82)."""
    if n_bins < 1:
        raise ValueError("invalid bin count")
    xs = as_index_series(x, _len_of(x))
    out = np.zeros(n_bins + 1, np.int64)
    L = _lib.load()
    if is_device(xs):
        import torch

        dev = xs.device or 0
        torch.cuda.current_stream(dev).synchronize()
        d = torch.empty(n_bins + 1, dtype=torch.int64, device=f"cuda:{dev}")
        ctx = _lib.context(dev)
        rc = L.tsds_op_equal_width_offsets(ctx.handle, xs.ptr, CODE[xs.dtype], length(xs), int(n_bins), d.data_ptr())
        _lib.check(rc, "equal_width_boundaries")
        out[:] = d.cpu().numpy()
    else:
        rc = L.tsds_host_equal_width_offsets(xs.ctypes.data, CODE[xs.dtype], length(xs), int(n_bins), out.ctypes.data)
        _lib.check(rc, "equal_width_boundaries")
    return out.astype(np.uint64)


def _len_of(x):
    if hasattr(x, "__cuda_array_interface__") or type(x).__module__.startswith("torch"):
        return int(x.shape[0]) if len(x.shape) else 0
    return np.asarray(x).shape[0]


def boundaries_parallel(x, length_, n_bins, workers):
    """Same boundaries as the sequential functions (binning.py:85-125)."""
    if n_bins < 1:
        raise ValueError("invalid bin count")
    if workers < 1:
        raise ValueError("invalid worker count")
    if x is None:
        return equal_count_boundaries(length_, n_bins)
    x = as_index_series(x, length_)
    return equal_width_boundaries(x if not is_device(x) else x.owner, n_bins)
