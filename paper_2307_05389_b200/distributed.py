"""Multi-GPU sharding (one process per GPU, torch.distributed for the plumbing).

Mirrors the reference's only parallel strategy -- contiguous bin chunks of
``ceil(n_bins / workers)`` handed to workers, outputs concatenated in bin
order (algorithms.py:82-100, binning.py:85-138) -- with ranks in place of
threads:

  * MinMax / M4: rank r scans bins [b0_r, b1_r) of its shard of y on its own
    GPU (tsds_downsample_bins_async), then the per-rank index lists are
    concatenated in rank order with an all-gather (NCCL over NVLink on GPUs,
    gloo in the CPU tests).  Bins are independent and emitted in bin order,
    so the result is bit-identical to the single-GPU call;
  * MinMaxLTTB: the preselection is sharded the same way over the sub-bins;
    the gathered candidates feed the (sequential) triangle stage, which
    every rank runs on identical inputs (replicated, no broadcast needed);
  * LTTB: replicas only (the walk is sequential);
  * batched MinMax: independent series partitioned across ranks.

Bin edges come from the reference's global formulas (equal-count, or the
exact equal-width searches on the host), so every rank agrees on them.
The per-rank compute is injectable (``compute=``) so the sharding logic is
tested on CPU with world_size 2 over gloo (tests/test_distributed_cpu.py).
"""

import ctypes

import numpy as np

from . import _lib
from .dtypes import CODE, as_index_series, as_value_series, length

WIDTH = {"minmax": 2, "m4": 4}


def shard_ranges(n_bins, world):
    """[(b0, b1)] per rank: contiguous chunks of ceil(n_bins / world) (algorithms.py:88-91)."""
    chunk = -(-n_bins // world)
    out = []
    for r in range(world):
        b0 = min(r * chunk, n_bins)
        out.append((b0, min(b0 + chunk, n_bins)))
    return out


def equal_count_offsets(length_, n_bins, add=0):
    k = np.arange(n_bins + 1, dtype=np.int64)
    return k * np.int64(length_) // np.int64(n_bins) + add


def host_offsets(x, length_, n_bins, add=0):
    """Bin offsets over x[0:length] (equal-width, uniform shortcut) or equal-count."""
    if x is None:
        return equal_count_offsets(length_, n_bins, add)
    L = _lib.load()
    out = np.zeros(n_bins + 1, np.int64)
    rc = L.tsds_host_equal_width_offsets(x.ctypes.data, CODE[x.dtype], length_, n_bins, out.ctypes.data)
    _lib.check(rc, "equal_width_offsets")
    return out + add


def is_uniform(x):
    return bool(_lib.load().tsds_host_is_uniform_spaced(x.ctypes.data, CODE[x.dtype], x.shape[0]))


def gpu_bins_compute(device):
    """Per-rank compute on `device`: (y_shard, off_rel, algo, base, nan) -> int64 indices."""

    def compute(y_shard, off_rel, algo, base, nan):
        import torch

        L = _lib.load()
        ctx = _lib.context(device)
        nb = off_rel.shape[0] - 1
        dev = f"cuda:{device}"
        yd = torch.from_numpy(np.ascontiguousarray(y_shard)).to(dev)
        od = torch.from_numpy(np.ascontiguousarray(off_rel, dtype=np.int64)).to(dev)
        out = torch.empty(WIDTH[algo] * nb, dtype=torch.int64, device=dev)
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        torch.cuda.current_stream(device).synchronize()
        rc = L.tsds_downsample_bins_async(
            ctx.handle, _lib.ALGO[algo], yd.data_ptr(), CODE[y_shard.dtype], od.data_ptr(), nb, int(base),
            1 if nan else 0, out.data_ptr(), cnt.data_ptr())
        _lib.check(rc, "downsample_bins")
        ctx.synchronize()
        return out[: int(cnt.item())].cpu().numpy()

    return compute


def allgather_varlen(local, group=None, device=None):
    """Concatenate every rank's int64 array in rank order (all-gather of padded buffers)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dev = torch.device("cpu") if device is None else torch.device("cuda", device)
    n = torch.tensor([local.shape[0]], dtype=torch.int64, device=dev)
    counts = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(counts, n, group=group)
    counts = [int(c.item()) for c in counts]
    cap = max(1, max(counts))
    buf = torch.zeros(cap, dtype=torch.int64, device=dev)
    buf[: local.shape[0]] = torch.from_numpy(np.ascontiguousarray(local, dtype=np.int64)).to(dev)
    parts = [torch.zeros(cap, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return np.concatenate([p[:c].cpu().numpy() for p, c in zip(parts, counts)])


def sharded_downsample(algo, *args, n_out, minmax_ratio=4, nan=False, group=None, device=None, compute=None,
                       stage2=None):
    """Sharded equivalent of ``downsample(algo, [x,] y, n_out=...)`` on every rank.

    Every rank passes the same host series; rank r scans its contiguous bin
    range on its GPU and the result (uint64, identical on all ranks) equals
    the single-GPU / reference result.
    """
    import torch.distributed as dist

    if algo not in ("minmax", "m4", "minmaxlttb", "lttb"):
        raise ValueError(f"unknown algorithm: {algo!r}")
    if len(args) == 1:
        x, y = None, args[0]
    elif len(args) == 2:
        x, y = args
    else:
        raise TypeError("expected positional arguments ([x,] y)")
    y = as_value_series(y)
    x = as_index_series(x, length(y))
    n = length(y)
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    if compute is None:
        compute = gpu_bins_compute(rank if device is None else device)

    if algo == "lttb":  # replicas only: the walk is sequential
        from . import algorithms

        return algorithms.lttb(x, y, n_out)
    if algo in WIDTH:
        w = WIDTH[algo]
        if n_out < w:
            raise ValueError("invalid n_out")
        if n_out % w:
            raise ValueError(f"n_out must be a multiple of {w}")
        if n == 0:
            raise ValueError("empty series")
        if n <= n_out:
            return np.arange(n, dtype=np.uint64)
        if x is not None and is_uniform(x):
            x = None
        nb = n_out // w
        off = host_offsets(x, n, nb)
        b0, b1 = shard_ranges(nb, world)[rank]
        local = np.zeros(0, np.int64)
        if b1 > b0:
            s, e = int(off[b0]), int(off[b1])
            local = compute(y[s:e], off[b0 : b1 + 1] - s, algo, s, nan)
        return allgather_varlen(local, group, device).astype(np.uint64)

    # minmaxlttb
    if n_out < 3:
        raise ValueError("n_out too small for LTTB")
    if minmax_ratio < 1:
        raise ValueError("invalid ratio")
    if n == 0:
        raise ValueError("empty series")
    from . import algorithms

    if n <= n_out * minmax_ratio:
        return algorithms.lttb(x, y, n_out)
    if x is not None and is_uniform(x):
        x = None
    nsub = (n_out - 2) * ((minmax_ratio + 1) // 2)
    off = host_offsets(None if x is None else x[1 : n - 1], n - 2, nsub, add=1)
    b0, b1 = shard_ranges(nsub, world)[rank]
    local = np.zeros(0, np.int64)
    if b1 > b0:
        s, e = int(off[b0]), int(off[b1])
        local = compute(y[s:e], off[b0 : b1 + 1] - s, "minmax", s, nan)
    sel = allgather_varlen(local, group, device)
    full = np.concatenate([[0], sel, [n - 1]]).astype(np.int64)
    m = full.shape[0]
    if m <= n_out:
        return full.astype(np.uint64)
    return (stage2 or lttb_stage2)(x, y, full, n_out)


def lttb_stage2(x, y, full, n_out):
    """The triangle stage over gathered candidates (tsds_lttb_stage2)."""
    L = _lib.load()
    y2 = np.ascontiguousarray(y[full])
    x2 = None if x is None else np.ascontiguousarray(x[full])
    out = np.zeros(n_out, np.int64)
    m2 = ctypes.c_int64(0)
    ctx = _lib.context()
    rc = L.tsds_lttb_stage2(
        ctx.handle, None if x2 is None else x2.ctypes.data, 0 if x2 is None else CODE[x2.dtype], y2.ctypes.data,
        CODE[y2.dtype], full.ctypes.data, full.shape[0], int(n_out), out.ctypes.data, ctypes.byref(m2))
    _lib.check(rc, "lttb_stage2")
    return out[: m2.value].astype(np.uint64)


def sharded_minmax_batched(Y, n_out, nan=False, group=None, device=None, compute=None):
    """Batched MinMax with the series partitioned across ranks (weak scaling).

    Returns (idx[S, n_out] uint64, counts[S]) on every rank.
    """
    import torch.distributed as dist
    from .algorithms import minmax_batched

    Y = np.asarray(Y)
    S = Y.shape[0]
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    s0, s1 = shard_ranges(S, world)[rank]
    if compute is None:
        def compute(block, n_out_, nan_):
            return minmax_batched(block, n_out_, nan=nan_)
    if s1 > s0:
        idx, cnt = compute(Y[s0:s1], n_out, nan)
        local = np.concatenate([cnt.astype(np.int64), idx.view(np.int64).reshape(-1)])
    else:
        local = np.zeros(0, np.int64)
    flat = allgather_varlen(local, group, device)
    idx = np.zeros((S, n_out), np.int64)
    counts = np.zeros(S, np.int64)
    pos = 0
    for r, (a, b) in enumerate(shard_ranges(S, world)):
        k = b - a
        if k <= 0:
            continue
        counts[a:b] = flat[pos : pos + k]
        pos += k
        idx[a:b] = flat[pos : pos + k * n_out].reshape(k, n_out)
        pos += k * n_out
    return idx.view(np.uint64), counts

