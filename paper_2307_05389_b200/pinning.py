"""Pin-on-reuse cache for large host inputs (extension; no reference counterpart).

A numpy array is pageable memory: every call has to stage it through pinned
slots (csrc/tsds_staging.h), which costs host-DRAM bandwidth (read + write +
DMA read) and tops out below the PCIe rate.  Downsampling is typically
called again and again on the same array (interactive zooming, different
n_out, the estimator classes), so the second time an array of at least
``TSDS_PIN_MIN_BYTES`` (default 64 MiB) is seen, its owner's buffer is
page-locked in place with ``tsds_host_register`` (cudaHostRegister,
~13 GB/s once) and later uploads are DMA'd directly from it at link speed.

Why not smaller arrays: on the pool's VMs the DMA rate from a registered
array depends on where the allocator placed it -- the same 40 MB series moved
at 23 GB/s in one process and 54 GB/s in another (transparent huge pages in
both, tools/thp_probe.py; the placement relative to the GPU's root complex is
not visible to the guest) -- against a steady 32-39 GB/s through the staging
ring, whose slots are driver-allocated.  From 64 MiB up the registered path
was at least on par with the ring (43-55 against 41-47 GB/s) and at the link
rate for multi-GB inputs (54.5 GB/s).

Safety: the registration is tied, through a weak reference, to the array at
the end of the ``.base`` chain -- the one that owns the memory or holds the
buffer export that keeps it mapped -- and is released when that array is
garbage collected, i.e. before the memory can be unmapped.  Arrays whose
memory lifetime cannot be tied to a numpy object (np.memmap, foreign array
interfaces) are never registered.  ``TSDS_PIN_CACHE`` = ``reuse`` (default) | ``always`` (pin
on first sight) | ``off``; ``TSDS_PIN_MAX_BYTES`` caps the pinned total
(default 1/4 of physical memory, least recently used evicted first).
"""

import os
import threading
import weakref
from collections import OrderedDict

import numpy as np

from . import _lib


def _default_cap():
    try:
        return os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") // 4
    except (ValueError, OSError, AttributeError):
        return 16 << 30


_mode = os.environ.get("TSDS_PIN_CACHE", "reuse").lower()
_min_bytes = int(os.environ.get("TSDS_PIN_MIN_BYTES", 64 << 20))
_max_bytes = int(os.environ.get("TSDS_PIN_MAX_BYTES", _default_cap()))
_lock = threading.Lock()
_seen = {}  # id(owner) -> sightings (negative: registration failed, do not retry)
_pinned = OrderedDict()  # id(owner) -> (ptr, nbytes, device)
_refs = {}  # id(owner) -> weakref keeping the bookkeeping in step with the owner's life
stats = {"registered": 0, "released": 0, "failed": 0, "hits": 0}


def configure(mode=None, min_bytes=None, max_bytes=None):
    """Change the policy at run time (also releases everything when mode == "off")."""
    global _mode, _min_bytes, _max_bytes
    if mode is not None:
        if mode not in ("reuse", "always", "off"):
            raise ValueError("mode must be 'reuse', 'always' or 'off'")
        _mode = mode
        if mode == "off":
            release_all()
    if min_bytes is not None:
        _min_bytes = int(min_bytes)
    if max_bytes is not None:
        _max_bytes = int(max_bytes)


def owner_of(a):
    """The ndarray at the end of a's ``.base`` chain if the memory cannot go
    away while that array is alive: it owns its data, or it wraps a
    buffer-protocol export (``np.frombuffer`` over an mmap / bytearray /
    bytes: the exporter refuses to close or resize while the export exists).
    None otherwise (np.memmap subclasses, foreign ``__array_interface__``
    objects, scalars)."""
    o = a
    while isinstance(o, np.ndarray) and isinstance(o.base, np.ndarray):
        o = o.base
    if type(o) is not np.ndarray:
        return None
    if o.flags.owndata or isinstance(o.base, memoryview):
        return o
    return None


def _release(key):
    ent = _pinned.pop(key, None)
    if ent is None:
        return
    ptr = ent[0]
    if ptr is None:  # already unregistered by the owner's finalizer
        return
    try:
        _lib.load().tsds_host_unregister(None, ptr)
        stats["released"] += 1
    except Exception:
        pass


_pending = []  # owners collected while the lock was held (a finalizer can run inside any allocation)


def _forget(key):
    _seen.pop(key, None)
    _refs.pop(key, None)
    _release(key)


def _on_collect(key):
    # The owner is gone: its pages must be released NOW, before the allocator can hand the same
    # addresses to a new array (a stale registration would DMA the old physical pages).  The
    # unregister needs no lock (nobody else can touch a dead owner's entry); only the
    # bookkeeping below may have to wait.
    ent = _pinned.get(key)
    if ent is not None and ent[0] is not None:
        _pinned[key] = (None, ent[1], ent[2])
        try:
            _lib.load().tsds_host_unregister(None, ent[0])
            stats["released"] += 1
        except Exception:
            pass
    if _lock.acquire(blocking=False):
        try:
            _forget(key)
        finally:
            _lock.release()
    else:  # this thread (or another) is inside the cache: handled at its next entry
        _pending.append(key)


def _drain_pending():
    while _pending:
        _forget(_pending.pop())


def release_all():
    with _lock:
        _drain_pending()
        for key in list(_pinned):
            _release(key)
        _seen.clear()


def pinned_bytes():
    return sum(e[1] for e in list(_pinned.values()) if e[0] is not None)


def note_host_input(a, device=None):
    """Called with every host array about to be handed to the library as
    TSDS_MEM_HOST.  Returns True when the array's memory is page-locked."""
    if _mode == "off" or not isinstance(a, np.ndarray) or a.nbytes < _min_bytes:
        return False
    o = owner_of(a)
    if o is None:
        return False
    key = id(o)
    with _lock:
        _drain_pending()
        if key in _pinned:
            _pinned.move_to_end(key)
            stats["hits"] += 1
            return True
        c = _seen.get(key, 0)
        if c < 0:
            return False
        if key not in _refs:
            r = weakref.finalize(o, _on_collect, key)
            r.atexit = False  # process teardown releases everything anyway
            _refs[key] = r
        _seen[key] = c + 1
        if _mode == "reuse" and c + 1 < 2:
            return False
        nbytes = o.nbytes
        if nbytes > _max_bytes:
            _seen[key] = -1
            return False
        while _pinned and pinned_bytes() + nbytes > _max_bytes:
            _release(next(iter(_pinned)))
        rc = _lib.load().tsds_host_register(_lib.context(device).handle, o.ctypes.data, nbytes)
        if rc != _lib.TSDS_OK:
            _seen[key] = -1
            stats["failed"] += 1
            return False
        _pinned[key] = (o.ctypes.data, nbytes, device)
        stats["registered"] += 1
        return True
