"""ctypes front-end of the CPU oracle (tsds_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's reference / cpu_baseline arm, never by the product package.
The oracle restates the reference `thinseries` path (scalar semantics,
SURVEY.md Appendix A); its parity with the real reference is pinned by
tests/test_oracle_golden.py against tests/golden/*.npz, which
tests/golden/make_golden.py produced by importing the reference itself.
"""

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")

DTYPE_CODES = {
    np.dtype(np.float16): 0,
    np.dtype(np.float32): 1,
    np.dtype(np.float64): 2,
    np.dtype(np.int8): 3,
    np.dtype(np.int16): 4,
    np.dtype(np.int32): 5,
    np.dtype(np.int64): 6,
    np.dtype(np.uint8): 7,
    np.dtype(np.uint16): 8,
    np.dtype(np.uint32): 9,
    np.dtype(np.uint64): 10,
}

ALGO_CODES = {"minmax": 1, "m4": 2, "lttb": 3, "minmaxlttb": 4}

_lib = None


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.or_argminmax.argtypes = [vp, i32, i64, i32, vp]
        L.or_equal_count.argtypes = [i64, i64, vp]
        L.or_is_uniform.argtypes = [vp, i32, i64]
        L.or_equal_width.argtypes = [vp, i32, i64, i64, vp]
        L.or_downsample.argtypes = [i32, vp, i32, vp, i32, i64, i64, i64, i32, i32, vp]
        L.or_downsample.restype = i64
        L.or_minmax_batched.argtypes = [vp, i32, i64, i64, i64, i32, i32, vp, vp]
        L.or_lttb_walk.argtypes = [vp, i32, vp, i32, i64, vp, i64, vp]
        L.or_lttb_walk.restype = i64
        L.or_lttb_near_ties.argtypes = [vp, i32, vp, i32, i64, vp, i64, ctypes.c_double, vp]
        L.or_lttb_near_ties.restype = i64
        L.or_fill_width_offsets.argtypes = [vp, i32, i64, ctypes.c_double, ctypes.c_double, i64, i64, i64, vp]
        L.or_bins_slots.argtypes = [vp, i32, vp, i64, i64, i32, i32, vp, vp]
        L.or_compact_bins.argtypes = [vp, vp, i32, i64, vp]
        L.or_compact_bins.restype = i64
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


def _x_view(x):
    if x is None:
        return None
    x = np.ascontiguousarray(x)
    if np.issubdtype(x.dtype, np.datetime64):
        x = x.view(np.int64)
    return x


def argminmax(y, nan=False):
    y = np.ascontiguousarray(y)
    out = np.zeros(2, np.int64)
    lib().or_argminmax(_ptr(y), DTYPE_CODES[y.dtype], y.shape[0], int(nan), _ptr(out))
    return int(out[0]), int(out[1])


def equal_count(length, n_bins):
    out = np.zeros(n_bins + 1, np.int64)
    lib().or_equal_count(length, n_bins, _ptr(out))
    return out.astype(np.uint64)


def is_uniform(x):
    x = _x_view(x)
    return bool(lib().or_is_uniform(_ptr(x), DTYPE_CODES[x.dtype], x.shape[0]))


def equal_width(x, n_bins):
    x = _x_view(x)
    out = np.zeros(n_bins + 1, np.int64)
    rc = lib().or_equal_width(_ptr(x), DTYPE_CODES[x.dtype], x.shape[0], n_bins, _ptr(out))
    if rc != 0:
        raise ValueError("invalid index span")
    return out.astype(np.uint64)


def downsample(algo, *args, n_out, minmax_ratio=4, nan=False, threads=1):
    """Indices of the reference algorithm on valid inputs (uint64)."""
    if len(args) == 1:
        x, y = None, args[0]
    else:
        x, y = args
    y = np.ascontiguousarray(y)
    x = _x_view(x)
    out = np.zeros(max(int(n_out), 1), np.int64)  # every algorithm returns <= n_out
    m = lib().or_downsample(
        ALGO_CODES[algo],
        _ptr(x),
        0 if x is None else DTYPE_CODES[x.dtype],
        _ptr(y),
        DTYPE_CODES[y.dtype],
        y.shape[0],
        int(n_out),
        int(minmax_ratio),
        int(nan),
        int(threads),
        _ptr(out),
    )
    if m == -2:
        raise ValueError("invalid index span")
    if m < 0:
        raise RuntimeError(f"oracle error {m}")
    return out[:m].astype(np.uint64)


def minmax_batched(Y, n_out, nan=False, threads=1):
    """Row s == downsample('minmax', Y[s], n_out); returns (idx[S, n_out], counts)."""
    Y = np.ascontiguousarray(Y)
    S, L = Y.shape
    out = np.zeros((S, n_out), np.int64)
    counts = np.zeros(S, np.int64)
    lib().or_minmax_batched(
        _ptr(Y), DTYPE_CODES[Y.dtype], S, L, int(n_out), int(nan), int(threads), _ptr(out), _ptr(counts)
    )
    return out.astype(np.uint64), counts


def lttb_walk(x, y, off):
    """The reference triangle walk with caller-supplied offsets (x None: implicit)."""
    y = np.ascontiguousarray(y)
    x = _x_view(x)
    off = np.ascontiguousarray(off, dtype=np.int64)
    out = np.zeros(off.shape[0] + 1, np.int64)
    m = lib().or_lttb_walk(_ptr(x), 0 if x is None else DTYPE_CODES[x.dtype], _ptr(y), DTYPE_CODES[y.dtype],
                           y.shape[0], _ptr(off), off.shape[0] - 1, _ptr(out))
    return out[:m]


def lttb_near_ties(x, y, off, rel=1e-12):
    """(count, bucket numbers) of the buckets whose two best triangle areas
    are within `rel` relative along the reference's own walk (sequential
    centroid sums, no FMA)."""
    y = np.ascontiguousarray(y)
    x = _x_view(x)
    off = np.ascontiguousarray(off, dtype=np.int64)
    buckets = np.zeros(max(off.shape[0] - 1, 1), np.int64)
    m = lib().or_lttb_near_ties(_ptr(x), 0 if x is None else DTYPE_CODES[x.dtype], _ptr(y), DTYPE_CODES[y.dtype],
                                y.shape[0], _ptr(off), off.shape[0] - 1, float(rel), _ptr(buckets))
    return int(m), buckets[:m]


def stage2(x, y, full, n_out):
    """MinMaxLTTB stage 2 on candidates `full` (algorithms.py:243-255)."""
    full = np.asarray(full, np.int64)
    m = full.shape[0]
    y2 = np.ascontiguousarray(y[full])
    nb = n_out - 2
    if x is None:
        off2 = (np.arange(nb + 1, dtype=np.int64) * (m - 2)) // nb + 1
        sel = lttb_walk(full, y2, off2)
    else:
        x2 = np.ascontiguousarray(np.asarray(x)[full])
        off2 = equal_width(x2[1:-1], nb).astype(np.int64) + 1
        sel = lttb_walk(x2, y2, off2)
    return full[sel].astype(np.uint64)


# --------------------------------------------------------------------------
# operator level (the reference numba kernels' own signatures)


def fill_width_offsets(x, x0, span, n_bins, k0, k1, out):
    """_kernels.fill_width_offsets: out[k] for k in [k0, k1)."""
    x = _x_view(x)
    lib().or_fill_width_offsets(_ptr(x), DTYPE_CODES[x.dtype], x.shape[0], float(x0), float(span), int(n_bins),
                                int(k0), int(k1), _ptr(out))


def bins_slots(width, y, off, b0, b1, idx, cnt, nan=False):
    """_kernels minmax_bins (width 2) / m4_bins (width 4) writing idx[width*b+t], cnt[b]."""
    y = np.ascontiguousarray(y)
    off = np.ascontiguousarray(off, dtype=np.int64)
    lib().or_bins_slots(_ptr(y), DTYPE_CODES[y.dtype], _ptr(off), int(b0), int(b1), int(width), int(nan), _ptr(idx),
                        _ptr(cnt))


def compact_bins(idx, cnt, width):
    """_kernels.compact_bins."""
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    cnt = np.ascontiguousarray(cnt, dtype=np.int64)
    out = np.zeros(max(1, int(cnt.sum())), np.int64)
    m = lib().or_compact_bins(_ptr(idx), _ptr(cnt), int(width), cnt.shape[0], _ptr(out))
    return out[:m]
