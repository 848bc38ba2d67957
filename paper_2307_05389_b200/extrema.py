"""Whole-series argmin/argmax and the ordinal transforms (mirrors thinseries.extrema).

`argminmax` runs the same streaming kernel as the downsamplers over a single
bin (extrema.py:142-155).  The reference's `argminmax_scalar` /
`argminmax_vector` select CPU code paths that are bit-identical for non-NaN
input; here both names are the one GPU kernel with the scalar path's
semantics (the reference's documented "reference path", extrema.py:111-124).
"""

import numpy as np

from . import _lib
from .algorithms import _context_for
from .dtypes import CODE, SIGNED_VIEW, as_value_series, is_device, length

_XOR_CONST = {
    np.dtype(np.int8): np.int8(-128),
    np.dtype(np.int16): np.int16(-32768),
    np.dtype(np.int32): np.int32(-2147483648),
    np.dtype(np.int64): np.int64(-9223372036854775808),
}
_UNSIGNED_VIEW = {v: k for k, v in SIGNED_VIEW.items()}


def ord_transform_i16(v):
    """f16 bit patterns (as int16) -> order-preserving int16 (extrema.py:38-47)."""
    v = np.asarray(v, dtype=np.int16)
    r = ((v >> 15) & np.int16(0x7FFF)) ^ v
    return r if r.ndim else np.int16(r)


def ord_transform_uint(v):
    """Unsigned ints -> order-preserving signed ints, an involution (extrema.py:53-68)."""
    a = np.asarray(v)
    if a.dtype in SIGNED_VIEW:
        signed = SIGNED_VIEW[a.dtype]
        r = a.view(signed) ^ _XOR_CONST[signed]
    elif a.dtype in _XOR_CONST:
        r = (a ^ _XOR_CONST[a.dtype]).view(_UNSIGNED_VIEW[a.dtype])
    else:
        raise ValueError("unsupported dtype")
    return r if a.ndim else r[()]


def argminmax(v, nan=False):
    """(argmin, argmax) of a whole series; first occurrence wins ties."""
    v = as_value_series(v)
    if length(v) == 0:
        raise ValueError("empty series")
    ctx, mem = _context_for(None, v)
    out = np.zeros(2, np.int64)
    rc = _lib.load().tsds_argminmax(
        ctx.handle,
        v.ptr if is_device(v) else v.ctypes.data,
        CODE[np.dtype(v.dtype)],
        length(v),
        1 if nan else 0,
        mem,
        out.ctypes.data,
    )
    _lib.check(rc, "argminmax")
    return int(out[0]), int(out[1])


def argminmax_scalar(v):
    return argminmax(v)


def argminmax_vector(v):
    return argminmax(v)


def nanargminmax(v):
    """(argmin, argmax) where any NaN wins both (first NaN)."""
    return argminmax(v, nan=True)

