"""ctypes binding of libtsds.so (include/tsds.h).

The shared library is built in-tree by ``python -m paper_2307_05389_b200.build``
(or ``__graft_entry__.build()``).  There is no CPU fallback: if the library
or a CUDA device is missing, calls fail loudly.  ctypes releases the GIL for
the duration of every foreign call, like the reference's ``nogil=True``
kernels (_kernels.py), so concurrent callers overlap.
"""

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TSDS_LIB") or os.path.join(HERE, "libtsds.so")

TSDS_OK = 0
TSDS_ERR_ARG = -1
TSDS_ERR_SPAN = -2
TSDS_ERR_CUDA = -3
TSDS_ERR_NOMEM = -4

ALGO = {"minmax": 1, "m4": 2, "lttb": 3, "minmaxlttb": 4}
MEM_HOST = 0
MEM_DEVICE = 1

EXPORTED = (
    "tsds_version",
    "tsds_set_option",
    "tsds_last_error",
    "tsds_device_count",
    "tsds_ctx_create",
    "tsds_ctx_destroy",
    "tsds_ctx_set_stream",
    "tsds_ctx_stream",
    "tsds_ctx_synchronize",
    "tsds_ctx_launches",
    "tsds_ctx_stat",
    "tsds_ctx_profile",
    "tsds_ctx_profile_read",
    "tsds_downsample",
    "tsds_downsample_async",
    "tsds_shard_bins_async",
    "tsds_shard_preselect_async",
    "tsds_records_concat",
    "tsds_lttb_stage2_async",
    "tsds_upload",
    "tsds_host_register",
    "tsds_host_unregister",
    "tsds_comm_unique_id",
    "tsds_comm_init",
    "tsds_comm_destroy",
    "tsds_comm_allgather",
    "tsds_minmax_batched",
    "tsds_minmax_batched_async",
    "tsds_argminmax",
    "tsds_op_is_uniform_spaced",
    "tsds_op_equal_count_offsets",
    "tsds_op_equal_width_offsets",
    "tsds_op_fill_width_offsets",
    "tsds_op_compact_bins",
    "tsds_op_minmax_bins",
    "tsds_op_m4_bins",
    "tsds_op_lttb",
    "tsds_host_is_uniform_spaced",
    "tsds_host_equal_width_offsets",
)

_lib = None
_lock = threading.Lock()
_tls = threading.local()


class TsdsError(RuntimeError):
    pass


def load():
    """Load libtsds.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2307_05389_b200.build` "
                "(there is no CPU fallback)"
            )
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        p64 = ctypes.POINTER(ctypes.c_int64)
        L.tsds_version.restype = i32
        L.tsds_last_error.restype = ctypes.c_char_p
        L.tsds_set_option.argtypes = [ctypes.c_char_p, i64]
        L.tsds_device_count.argtypes = [ctypes.POINTER(ctypes.c_int)]
        L.tsds_ctx_create.argtypes = [i32, ctypes.POINTER(vp)]
        L.tsds_ctx_destroy.argtypes = [vp]
        L.tsds_ctx_destroy.restype = None
        L.tsds_ctx_set_stream.argtypes = [vp, vp]
        L.tsds_ctx_stream.argtypes = [vp]
        L.tsds_ctx_stream.restype = vp
        L.tsds_ctx_synchronize.argtypes = [vp]
        L.tsds_ctx_launches.argtypes = [vp]
        L.tsds_ctx_launches.restype = i64
        L.tsds_ctx_stat.argtypes = [vp, ctypes.c_char_p]
        L.tsds_ctx_stat.restype = i64
        L.tsds_ctx_profile.argtypes = [vp, i32]
        L.tsds_ctx_profile_read.argtypes = [vp, ctypes.POINTER(ctypes.c_double), p64]
        L.tsds_downsample.argtypes = [vp, i32, vp, i32, vp, i32, i64, i64, i64, i32, i32, vp, p64]
        L.tsds_downsample_async.argtypes = [vp, i32, vp, i32, vp, i32, i64, i64, i64, i32, vp, vp, vp]
        L.tsds_shard_bins_async.argtypes = [vp, i32, vp, i32, vp, i64, i64, i64, i64, i32, i32, vp]
        L.tsds_shard_preselect_async.argtypes = [vp, vp, i32, vp, i32, vp, i64, i64, i64, i64, i32, i32, i64, i64, i64,
                                                 vp]
        L.tsds_records_concat.argtypes = [vp, vp, i32, i64, i32, vp, i64, vp]
        L.tsds_lttb_stage2_async.argtypes = [vp, vp, i64, vp, i32, vp, i32, i64, vp, vp]
        L.tsds_upload.argtypes = [vp, vp, vp, i64]
        L.tsds_host_register.argtypes = [vp, vp, i64]
        L.tsds_host_unregister.argtypes = [vp, vp]
        L.tsds_comm_unique_id.argtypes = [vp]
        L.tsds_comm_init.argtypes = [vp, i32, i32, vp, ctypes.POINTER(vp)]
        L.tsds_comm_destroy.argtypes = [vp]
        L.tsds_comm_destroy.restype = None
        L.tsds_comm_allgather.argtypes = [vp, vp, vp, i64]
        L.tsds_minmax_batched.argtypes =[vp, vp, i32, i64, i64, i64, i32, i32, vp, vp]
        L.tsds_minmax_batched_async.argtypes = [vp, vp, i32, i64, i64, i64, i32, vp, vp]
        L.tsds_argminmax.argtypes = [vp, vp, i32, i64, i32, i32, vp]
        L.tsds_op_is_uniform_spaced.argtypes = [vp, vp, i32, i64, vp]
        L.tsds_op_equal_count_offsets.argtypes = [vp, i64, i64, vp]
        L.tsds_op_equal_width_offsets.argtypes = [vp, vp, i32, i64, i64, vp]
        L.tsds_op_fill_width_offsets.argtypes = [vp, vp, i32, i64, ctypes.c_double, ctypes.c_double, i64, i64, i64,
                                                 vp]
        L.tsds_op_compact_bins.argtypes = [vp, vp, vp, i32, i64, vp, vp]
        L.tsds_op_minmax_bins.argtypes = [vp, vp, i32, vp, i64, i64, i32, vp, vp]
        L.tsds_op_m4_bins.argtypes = [vp, vp, i32, vp, i64, i64, i32, vp, vp]
        L.tsds_op_lttb.argtypes = [vp, vp, vp, i32, i64, vp, i64, vp, p64]
        L.tsds_host_is_uniform_spaced.argtypes = [vp, i32, i64]
        L.tsds_host_equal_width_offsets.argtypes = [vp, i32, i64, i64, vp]
        for name in EXPORTED:
            getattr(L, name)  # every declared symbol must resolve
        _lib = L
    return _lib


def last_error():
    return load().tsds_last_error().decode(errors="replace")


def check(rc, what=""):
    if rc == TSDS_OK:
        return
    msg = last_error()
    if rc == TSDS_ERR_SPAN:
        raise ValueError("invalid index span")
    if rc == TSDS_ERR_ARG:
        raise ValueError(msg or f"{what}: invalid argument")
    if rc == TSDS_ERR_NOMEM:
        raise MemoryError(msg or f"{what}: out of device memory")
    raise TsdsError(f"{what}: {msg}")


def device_count():
    n = ctypes.c_int(0)
    load().tsds_device_count(ctypes.byref(n))
    return n.value


class Context:
    """One libtsds context (CUDA stream + device workspace) per thread and device."""

    def __init__(self, device):
        L = load()
        h = ctypes.c_void_p()
        rc = L.tsds_ctx_create(int(device), ctypes.byref(h))
        if rc != TSDS_OK:
            raise TsdsError(f"cannot create a CUDA context on device {device}: {last_error()}")
        self.handle = h
        self.device = int(device)

    def __del__(self):
        try:
            if self.handle and _lib is not None:
                _lib.tsds_ctx_destroy(self.handle)
        except Exception:
            pass
        self.handle = None

    @property
    def stream(self):
        return load().tsds_ctx_stream(self.handle)

    def set_stream(self, stream_ptr):
        load().tsds_ctx_set_stream(self.handle, stream_ptr)

    def synchronize(self):
        check(load().tsds_ctx_synchronize(self.handle), "synchronize")

    @property
    def launches(self):
        return int(load().tsds_ctx_launches(self.handle))


def upload(ctx, dst_tensor, src_array):
    """Copy a contiguous host array into a device tensor on ctx's stream
    (staging ring for pageable memory); synchronises before returning."""
    check(load().tsds_upload(ctx.handle, dst_tensor.data_ptr(), src_array.ctypes.data, src_array.nbytes), "upload")
    ctx.synchronize()


def context(device=None):
    """Thread-local context for `device` (default: current torch device or 0)."""
    if device is None:
        device = getattr(_tls, "default_device", 0)
    cache = getattr(_tls, "ctxs", None)
    if cache is None:
        cache = _tls.ctxs = {}
    c = cache.get(device)
    if c is None:
        c = cache[device] = Context(device)
    return c


def set_default_device(device):
    _tls.default_device = int(device)
