"""The downsampling algorithms on the B200 (mirrors thinseries.algorithms).

Validation order, identity rule and error strings follow the reference
(algorithms.py:108-255).  The work itself is one call into libtsds.so per
invocation: the device pipeline does binning, the per-bin argmin/argmax
scan, compaction and (for the LTTB family) the triangle walk.  `parallel`
and `workers` are accepted for interface parity and never change the
output -- the GPU path is always parallel (the reference proves its own
parallel runs bit-identical to sequential ones, test_acceptance.py:179-201).
`workers` is still validated exactly where the reference validates it.
"""

import ctypes
import os

import numpy as np

from . import _lib
from .dtypes import CODE, is_device, length


def _identity(n):
    return np.arange(n, dtype=np.uint64)


def _resolve_workers(workers):
    if workers is None:
        return os.cpu_count() or 1
    if workers < 1:
        raise ValueError("invalid worker count")
    return workers


def _check_not_empty(y):
    if length(y) == 0:
        raise ValueError("empty series")


def every_nth(length_, n_out):
    """Stride selection (algorithms.py:108-115); index arithmetic only."""
    if n_out < 1:
        raise ValueError("invalid n_out")
    if length_ <= n_out:
        return _identity(length_)
    stride = -(-length_ // n_out)
    return np.arange(0, length_, stride, dtype=np.uint64)


def _ptr(a):
    if a is None:
        return None
    if is_device(a):
        return a.ptr
    return a.ctypes.data


def _context_for(x, y):
    dev_y = is_device(y)
    dev_x = x is not None and is_device(x)
    if x is not None and dev_x != dev_y:
        raise TypeError("x and y must both be host arrays or both device arrays")
    if dev_y:
        dev = y.device
        if dev is None:
            dev = 0
        try:
            import torch

            torch.cuda.current_stream(dev).synchronize()
        except Exception:
            pass
        return _lib.context(dev), _lib.MEM_DEVICE
    from . import pinning

    pinning.note_host_input(y)
    return _lib.context(), _lib.MEM_HOST


def _run(algo, x, y, n_out, ratio=4, nan=False):
    """One tsds_downsample call; x must already be validated."""
    ctx, mem = _context_for(x, y)
    out = np.empty(max(int(n_out), 1), np.int64)
    m = ctypes.c_int64(0)
    rc = _lib.load().tsds_downsample(
        ctx.handle,
        _lib.ALGO[algo],
        _ptr(x),
        0 if x is None else CODE[np.dtype(x.dtype)],
        _ptr(y),
        CODE[np.dtype(y.dtype)],
        length(y),
        int(n_out),
        int(ratio),
        1 if nan else 0,
        mem,
        out.ctypes.data,
        ctypes.byref(m),
    )
    _lib.check(rc, algo)
    return out[: m.value].view(np.uint64)


def minmax(x, y, n_out, parallel=False, workers=None, nan=False):
    """Per bin: positions of the minimum and maximum value (algorithms.py:118-145)."""
    if n_out < 2:
        raise ValueError("invalid n_out")
    if n_out % 2:
        raise ValueError("n_out must be a multiple of 2")
    _check_not_empty(y)
    if length(y) <= n_out:
        return _identity(length(y))
    _resolve_workers(workers)
    return _run("minmax", x, y, n_out, nan=nan)


def m4(x, y, n_out, parallel=False, workers=None, nan=False):
    """Per bin: first, argmin, argmax, last -- sorted, deduplicated (algorithms.py:148-175)."""
    if n_out < 4:
        raise ValueError("invalid n_out")
    if n_out % 4:
        raise ValueError("n_out must be a multiple of 4")
    _check_not_empty(y)
    if length(y) <= n_out:
        return _identity(length(y))
    _resolve_workers(workers)
    return _run("m4", x, y, n_out, nan=nan)


def lttb(x, y, n_out, parallel=False, workers=None):
    """Largest-triangle selection over n_out-2 interior bins (algorithms.py:184-208)."""
    if n_out < 3:
        raise ValueError("n_out too small for LTTB")
    _check_not_empty(y)
    if length(y) <= n_out:
        return _identity(length(y))
    return _run("lttb", x, y, n_out)


def minmaxlttb(x, y, n_out, ratio=4, parallel=False, workers=None, nan=False):
    """Two-stage LTTB: MinMax preselection, then the triangle pass (algorithms.py:211-255)."""
    if n_out < 3:
        raise ValueError("n_out too small for LTTB")
    if ratio < 1:
        raise ValueError("invalid ratio")
    _check_not_empty(y)
    if length(y) <= n_out * ratio:
        return lttb(x, y, n_out, parallel=parallel, workers=workers)
    _resolve_workers(workers)
    return _run("minmaxlttb", x, y, n_out, ratio=ratio, nan=nan)


def minmax_batched(Y, n_out, nan=False):
    """MinMax over every row of a 2-D batch (extension).

    Returns (idx, counts): idx is uint64[S, n_out] whose row s holds
    ``counts[s]`` valid indices equal to ``minmax(None, Y[s], n_out)``.
    """
    if n_out < 2:
        raise ValueError("invalid n_out")
    if n_out % 2:
        raise ValueError("n_out must be a multiple of 2")
    dev = None
    mod = type(Y).__module__
    if mod.startswith("torch"):
        import torch

        if isinstance(Y, torch.Tensor) and Y.is_cuda:
            from .dtypes import _torch_dtype_map

            npdt = _torch_dtype_map().get(Y.dtype)
            if npdt is None:
                raise ValueError("unsupported dtype")
            if Y.dim() != 2:
                raise ValueError("expected a 2-D batch")
            if not Y.is_contiguous():
                raise ValueError("non-contiguous input")
            torch.cuda.current_stream(Y.device).synchronize()
            dev = Y.device.index or 0
            S, L = Y.shape
            ptr, dt = Y.data_ptr(), np.dtype(npdt)
    if dev is None:
        Y = np.asarray(Y)
        if Y.dtype not in CODE:
            raise ValueError("unsupported dtype")
        if Y.ndim != 2:
            raise ValueError("expected a 2-D batch")
        if not Y.flags.c_contiguous:
            raise ValueError("non-contiguous input")
        S, L = Y.shape
        ptr, dt = Y.ctypes.data, Y.dtype
    if L == 0:
        raise ValueError("empty series")
    out = np.zeros((S, n_out), np.int64)
    counts = np.zeros(S, np.int64)
    if S == 0:
        return out.view(np.uint64), counts
    ctx = _lib.context(0 if dev is None else dev)
    if dev is None:
        from . import pinning

        pinning.note_host_input(Y)
    rc = _lib.load().tsds_minmax_batched(
        ctx.handle,
        ptr,
        CODE[dt],
        int(S),
        int(L),
        int(n_out),
        1 if nan else 0,
        _lib.MEM_HOST if dev is None else _lib.MEM_DEVICE,
        out.ctypes.data,
        counts.ctypes.data,
    )
    _lib.check(rc, "minmax_batched")
    return out.view(np.uint64), counts
