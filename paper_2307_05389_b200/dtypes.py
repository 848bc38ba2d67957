"""Element types and input validation (mirrors thinseries.dtypes, dtypes.py:1-80).

Accepts numpy arrays (host memory) and CUDA device arrays (torch tensors or
anything exposing ``__cuda_array_interface__``).  Error strings and check
order are the reference's, so callers see identical exceptions.
"""

import numpy as np

VALUE_DTYPES = {
    "f16": np.dtype(np.float16),
    "f32": np.dtype(np.float32),
    "f64": np.dtype(np.float64),
    "i8": np.dtype(np.int8),
    "i16": np.dtype(np.int16),
    "i32": np.dtype(np.int32),
    "i64": np.dtype(np.int64),
    "u8": np.dtype(np.uint8),
    "u16": np.dtype(np.uint16),
    "u32": np.dtype(np.uint32),
    "u64": np.dtype(np.uint64),
}
TAG_BY_DTYPE = {dt: tag for tag, dt in VALUE_DTYPES.items()}
# dtype code of the C ABI (include/tsds.h)
CODE = {dt: i for i, dt in enumerate(VALUE_DTYPES.values())}

SIGNED_VIEW = {
    np.dtype(np.uint8): np.dtype(np.int8),
    np.dtype(np.uint16): np.dtype(np.int16),
    np.dtype(np.uint32): np.dtype(np.int32),
    np.dtype(np.uint64): np.dtype(np.int64),
}


def tag_of(arr):
    try:
        return TAG_BY_DTYPE[np.dtype(arr.dtype)]
    except (KeyError, TypeError):
        raise ValueError("unsupported dtype") from None


class DeviceSeries:
    """A 1-D CUDA array seen through __cuda_array_interface__ (zero-copy)."""

    __slots__ = ("ptr", "dtype", "shape", "device", "owner")

    def __init__(self, ptr, dtype, shape, device, owner):
        self.ptr = ptr
        self.dtype = dtype
        self.shape = shape
        self.device = device
        self.owner = owner  # keeps the producer alive

    @property
    def ndim(self):
        return len(self.shape)

    @property
    def nbytes(self):
        return int(np.prod(self.shape)) * self.dtype.itemsize


def _torch_dtype_map():
    import torch

    m = {
        torch.float16: np.float16,
        torch.float32: np.float32,
        torch.float64: np.float64,
        torch.int8: np.int8,
        torch.int16: np.int16,
        torch.int32: np.int32,
        torch.int64: np.int64,
        torch.uint8: np.uint8,
    }
    for name, npdt in (("uint16", np.uint16), ("uint32", np.uint32), ("uint64", np.uint64)):
        if hasattr(torch, name):
            m[getattr(torch, name)] = npdt
    return m


def _as_device(obj):
    """DeviceSeries for CUDA arrays, None for host objects."""
    if isinstance(obj, DeviceSeries):
        return obj
    mod = type(obj).__module__
    if mod.startswith("torch"):
        import torch

        if isinstance(obj, torch.Tensor) and obj.is_cuda:
            npdt = _torch_dtype_map().get(obj.dtype)
            if npdt is None:
                raise ValueError("unsupported dtype")
            if obj.dim() != 1:
                raise ValueError("expected a 1-D series")
            if not obj.is_contiguous():
                raise ValueError("non-contiguous input")
            return DeviceSeries(obj.data_ptr(), np.dtype(npdt), tuple(obj.shape), obj.device.index or 0, obj)
        return None
    cai = getattr(obj, "__cuda_array_interface__", None)
    if cai is None:
        return None
    dt = np.dtype(cai["typestr"])
    shape = tuple(cai["shape"])
    if dt not in TAG_BY_DTYPE:
        raise ValueError("unsupported dtype")
    if len(shape) != 1:
        raise ValueError("expected a 1-D series")
    strides = cai.get("strides")
    if strides is not None and shape and shape[0] > 1 and strides[0] != dt.itemsize:
        raise ValueError("non-contiguous input")
    return DeviceSeries(int(cai["data"][0]), dt, shape, None, obj)


def as_value_series(y):
    """Validate y as a 1-D contiguous series of a supported dtype (dtypes.py:44-57)."""
    d = _as_device(y)
    if d is not None:
        return d
    y = np.asarray(y)
    if y.dtype not in TAG_BY_DTYPE:
        raise ValueError("unsupported dtype")
    if y.ndim != 1:
        raise ValueError("expected a 1-D series")
    if not y.flags.c_contiguous:
        raise ValueError("non-contiguous input")
    return y


def as_index_series(x, length):
    """Validate optional x against its value series (dtypes.py:60-80)."""
    if x is None:
        return None
    d = _as_device(x)
    if d is not None:
        if d.dtype == np.float16:
            raise ValueError("unsupported dtype")
        if d.shape[0] != length:
            raise ValueError("length mismatch")
        return d
    x = np.asarray(x)
    if np.issubdtype(x.dtype, np.datetime64):
        x = x.view(np.int64)
    if x.dtype not in TAG_BY_DTYPE or x.dtype == np.float16:
        raise ValueError("unsupported dtype")
    if x.ndim != 1:
        raise ValueError("expected a 1-D series")
    if not x.flags.c_contiguous:
        raise ValueError("non-contiguous input")
    if x.shape[0] != length:
        raise ValueError("length mismatch")
    return x


def is_device(a):
    return isinstance(a, DeviceSeries)


def length(a):
    return int(a.shape[0])
