"""Multi-GPU sharding: one process per GPU, device-resident shards.

The reference has one parallel strategy: contiguous bin chunks of
``ceil(n_bins / workers)`` handed to workers, outputs concatenated in bin
order (``_run_bins``, algorithms.py:82-100; ``boundaries_parallel``,
binning.py:85-138).  Here the workers are ranks:

  * a ShardPlan -- computed identically on every rank from the global bin
    edges (equal-count formula, or the reference's exact equal-width search
    over the host x: O(n_bins log n) probes) -- gives rank r the bins
    [b0_r, b1_r) and the element span [e0_r, e1_r) it must hold;
  * rank r keeps only y[e0_r:e1_r] (and x[e0_r:e1_r] for MinMaxLTTB) in its
    HBM (ShardedSeries); a step scans its bins on its GPU and writes one
    fixed-size record (include/tsds.h, "Sharded path");
  * the records are all-gathered over NCCL by the library's communicator
    (tsds_comm_*, NVLink/NVSwitch) and concatenated on the device in rank
    order, i.e. bin order: bit-identical to the single-GPU result;
  * MinMax / M4: the concatenation is the result;
  * MinMaxLTTB: the records carry each candidate's raw x / y bits, so every
    rank runs the (sequential, ~2*n_out-point) triangle stage on its own
    GPU (tsds_lttb_stage2_async) -- replicated, no broadcast needed;
  * LTTB: replicas only (the walk is sequential);
  * batched MinMax: the series are partitioned across ranks, no exchange
    beyond gathering the per-series results.

The per-rank compute is a backend object (GpuBackend here); tests swap in
a CPU oracle backend to check the plan, record layout, exchange and
ordering logic with world_size 2 over gloo (tests/test_distributed_cpu.py).
"""

import ctypes
from dataclasses import dataclass, field

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
    """binning.py:27-40: floor(k * len / n_bins) (+ add)."""
    k = np.arange(n_bins + 1, dtype=np.int64)
    return k * np.int64(length_) // np.int64(n_bins) + add


def host_offsets(x, length_, n_bins, add=0):
    """Bin offsets over x[0:length] (equal-width with the uniform shortcut) or equal-count."""
    if x is None:
        return equal_count_offsets(length_, n_bins, add)
    L = _lib.load()
    out = np.zeros(n_bins + 1, np.int64)
    rc = L.tsds_host_equal_width_offsets(x.ctypes.data, CODE[x.dtype], length_, n_bins, out.ctypes.data)
    _lib.check(rc, "equal_width_offsets")
    return out + add


def is_uniform(x):
    """is_uniform_spaced (_kernels.py:506-518) with the reference's arithmetic typing."""
    return bool(_lib.load().tsds_host_is_uniform_spaced(x.ctypes.data, CODE[x.dtype], x.shape[0]))


def _torch_dtype(dt):
    import torch

    return {np.dtype(np.float16): torch.float16, np.dtype(np.float32): torch.float32,
            np.dtype(np.float64): torch.float64, np.dtype(np.int8): torch.int8, np.dtype(np.int16): torch.int16,
            np.dtype(np.int32): torch.int32, np.dtype(np.int64): torch.int64, np.dtype(np.uint8): torch.uint8,
            np.dtype(np.uint16): torch.uint16, np.dtype(np.uint32): torch.uint32,
            np.dtype(np.uint64): torch.uint64}[np.dtype(dt)]


# ---------------------------------------------------------------------------- plan


@dataclass
class ShardPlan:
    """How one series is split across `world` ranks (identical on every rank)."""

    algo: str                 # "minmax" | "m4" | "minmaxlttb" (sharded) | "identity" | "lttb" (replicas)
    n: int
    n_out: int
    world: int
    off: np.ndarray = None    # global offsets of the (sub-)bins, absolute element indices
    ranges: list = field(default_factory=list)   # [(b0, b1)] bins per rank
    spans: list = field(default_factory=list)    # [(e0, e1)] elements each rank holds
    monotone: bool = True
    x_used: bool = False      # x takes part (False: absent or uniform -> dropped, api.py:19-28)
    cap: int = 0              # record entries per rank
    nfields: int = 1
    ratio: int = 4

    def scan_span(self, rank):
        """(relative offsets, span_begin, span_end) of rank's bins inside its shard."""
        b0, b1 = self.ranges[rank]
        e0 = self.spans[rank][0]
        rel = self.off[b0 : b1 + 1] - e0
        if b1 == b0:
            return rel, 0, 0
        if self.monotone:
            return rel, int(rel[0]), int(rel[-1])
        return rel, int(rel.min()), int(rel.max())


def _element_span(off, b0, b1, monotone):
    if b1 == b0:
        return 0, 0
    seg = off[b0 : b1 + 1]
    if monotone:
        return int(seg[0]), int(seg[-1])
    return int(seg.min()), int(seg.max())


def make_plan(algo, x, n, n_out, minmax_ratio=4, world=1):
    """Validation (same order and messages as algorithms.py) + the shard layout."""
    if algo in WIDTH:
        w = WIDTH[algo]
        if n_out < w:
            raise ValueError("invalid n_out")
        if n_out % w:
            raise ValueError(f"n_out must be a multiple of {w}")
        if n == 0:
            raise ValueError("empty series")
        if n <= n_out:
            return ShardPlan("identity", n, n_out, world)
        if x is not None and is_uniform(x):
            x = None
        nb = n_out // w
        off = host_offsets(x, n, nb)
        mono = bool(np.all(off[1:] >= off[:-1]))
        ranges = shard_ranges(nb, world)
        spans = [_element_span(off, b0, b1, mono) for b0, b1 in ranges]
        cap = w * max(1, max(b1 - b0 for b0, b1 in ranges))
        return ShardPlan(algo, n, n_out, world, off, ranges, spans, mono, x is not None, cap, 1)
    if algo == "minmaxlttb":
        if n_out < 3:
            raise ValueError("n_out too small for LTTB")
        if minmax_ratio < 1:
            raise ValueError("invalid ratio")
        if n == 0:
            raise ValueError("empty series")
        if n <= n_out:
            return ShardPlan("identity", n, n_out, world)
        if n <= n_out * minmax_ratio:
            return ShardPlan("lttb", n, n_out, world, ratio=minmax_ratio)
        if x is not None and is_uniform(x):
            x = None
        nsub = (n_out - 2) * ((minmax_ratio + 1) // 2)
        off = host_offsets(None if x is None else x[1 : n - 1], n - 2, nsub, add=1)
        mono = bool(np.all(off[1:] >= off[:-1]))
        ranges = shard_ranges(nsub, world)
        spans = []
        for r, (b0, b1) in enumerate(ranges):
            e0, e1 = _element_span(off, b0, b1, mono) if b1 > b0 else (None, None)
            if r == 0:  # the first rank owns frame point 0 (algorithms.py:237)
                e0, e1 = 0, max(e1 or 1, 1)
            if r == world - 1:  # the last rank owns frame point n-1
                e0 = n - 1 if e0 is None else min(e0, n - 1)
                e1 = n
            spans.append((0, 0) if e0 is None else (e0, e1))
        cap = 2 * max(1, max(b1 - b0 for b0, b1 in ranges)) + 2
        return ShardPlan("minmaxlttb", n, n_out, world, off, ranges, spans, mono, x is not None, cap, 3,
                         minmax_ratio)
    if algo == "lttb":
        if n_out < 3:
            raise ValueError("n_out too small for LTTB")
        if n == 0:
            raise ValueError("empty series")
        return ShardPlan("identity" if n <= n_out else "lttb", n, n_out, world)
    raise ValueError(f"unknown algorithm: {algo!r}")


# ------------------------------------------------------------------ exchanges


class NcclExchange:
    """All-gather through the library's communicator (tsds_comm_*: NCCL over
    NVLink/NVSwitch, on the context's stream).  The 128-byte NCCL id is made
    by rank 0 and broadcast over the torch.distributed process group."""

    def __init__(self, ctx, group=None):
        import torch.distributed as dist

        L = _lib.load()
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        uid = ctypes.create_string_buffer(128)
        if self.rank == 0:
            _lib.check(L.tsds_comm_unique_id(uid), "comm_unique_id")
        box = [uid.raw if self.rank == 0 else None]
        dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        uid = ctypes.create_string_buffer(box[0], 128)
        h = ctypes.c_void_p()
        _lib.check(L.tsds_comm_init(ctx.handle, self.world, self.rank, uid, ctypes.byref(h)), "comm_init")
        self.handle = h
        self.ctx = ctx

    def allgather(self, send, recv):
        """send: device tensor; recv: device tensor of world * send.numel() (enqueued, no sync)."""
        _lib.check(_lib.load().tsds_comm_allgather(self.handle, send.data_ptr(), recv.data_ptr(),
                                                   send.numel() * send.element_size()), "comm_allgather")

    def close(self):
        if getattr(self, "handle", None):
            _lib.load().tsds_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class TorchExchange:
    """All-gather over a torch.distributed group (any backend; gloo moves the
    records through host memory).  Used when NCCL is not the group's backend."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.group = group
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)

    def allgather(self, send, recv):
        import torch
        import torch.distributed as dist

        if send.is_cuda:  # the record was written on the library's stream
            torch.cuda.synchronize(send.device)
        parts = [torch.empty_like(send, device="cpu") for _ in range(self.world)]
        dist.all_gather(parts, send.cpu(), group=self.group)
        recv.copy_(torch.cat(parts).to(recv.device))
        if recv.is_cuda:  # visible to the library's stream before its next kernel
            torch.cuda.synchronize(recv.device)

    def close(self):
        pass


def default_exchange(ctx, group=None):
    import torch.distributed as dist

    return NcclExchange(ctx, group) if dist.get_backend(group) == "nccl" else TorchExchange(group)


# ------------------------------------------------------------------- backend


class GpuBackend:
    """The rank's device work through the C ABI (libtsds.so); everything is
    enqueued on the context's stream (no host synchronisation inside a step)."""

    def __init__(self, device):
        self.device = int(device)
        self.L = _lib.load()
        self.ctx = _lib.context(self.device)

    def shard_record(self, plan, rank, y_dev, ydt, x_dev, xdt, off_dev, rec, nan):
        b0, b1 = plan.ranges[rank]
        rel, s0, s1 = plan.scan_span(rank)
        e0 = plan.spans[rank][0]
        if plan.algo in WIDTH:
            if b1 == b0:
                rec.zero_()
                return
            _lib.check(self.L.tsds_shard_bins_async(self.ctx.handle, _lib.ALGO[plan.algo], y_dev.data_ptr(), ydt,
                                                    off_dev.data_ptr(), b1 - b0, e0, s0, s1, int(plan.monotone),
                                                    int(nan), rec.data_ptr()), "shard_bins")
            return
        first = 0 if rank == 0 else -1
        last = plan.n - 1 if rank == plan.world - 1 else -1
        _lib.check(self.L.tsds_shard_preselect_async(
            self.ctx.handle, y_dev.data_ptr(), ydt, None if x_dev is None else x_dev.data_ptr(), xdt,
            off_dev.data_ptr(), b1 - b0, e0, s0, s1, int(plan.monotone), int(nan), first, last, plan.cap,
            rec.data_ptr()), "shard_preselect")

    def concat(self, recv, world, cap, nf, out, ld_out, count):
        _lib.check(self.L.tsds_records_concat(self.ctx.handle, recv.data_ptr(), world, cap, nf, out.data_ptr(), ld_out,
                                              count.data_ptr()), "records_concat")

    def stage2(self, plan, cand, xbits, xdt, ybits, ydt, out, count):
        _lib.check(self.L.tsds_lttb_stage2_async(self.ctx.handle, cand.data_ptr(), plan.cap * plan.world,
                                                 None if xbits is None else xbits.data_ptr(), xdt, ybits.data_ptr(),
                                                 ydt, plan.n_out, out.data_ptr(), count.data_ptr()), "lttb_stage2")

    def batched_block(self, y_dev, ydt, nrows, L, n_out, nan, blk, rows):
        """Rows of a batch into blk = [counts(rows) | idx(rows * n_out)]."""
        if nrows == 0:
            blk.zero_()
            return
        _lib.check(self.L.tsds_minmax_batched_async(self.ctx.handle, y_dev.data_ptr(), ydt, nrows, L, n_out, int(nan),
                                                    blk[rows:].data_ptr(), blk[:rows].data_ptr()), "minmax_batched")

    def synchronize(self):
        self.ctx.synchronize()


# -------------------------------------------------------------- sharded series


class ShardedSeries:
    """Rank `rank`'s device-resident shard of one series under `plan`.

    ``step()`` enqueues one sharded downsample (shard scan -> record ->
    all-gather -> rank-order concatenation -> [MinMaxLTTB: triangle stage])
    on the rank's stream; ``result()`` synchronises and returns the uint64
    indices, identical on every rank and equal to the single-GPU call.
    """

    def __init__(self, plan, rank, y_shard, x_shard=None, exchange=None, backend=None, nan=False, dtypes=None,
                 x_host=None):
        import torch

        self.plan, self.rank, self.nan = plan, rank, nan
        # MinMaxLTTB with x kept on the host: the ~2*n_bins candidates' x bits are
        # gathered there after the scan instead of shipping the whole x shard
        self.x_host = x_host if plan.x_used and x_shard is None else None
        self.backend = backend
        self.exchange = exchange
        self.y = y_shard
        self.x = x_shard if plan.x_used else None
        self.ydt, self.xdt = dtypes if dtypes is not None else (0, 0)
        dev = y_shard.device
        nf, cap, world = plan.nfields, max(plan.cap, 1), plan.world
        self.rec = torch.zeros(1 + nf * cap, dtype=torch.int64, device=dev)
        self.recv = torch.zeros(world * (1 + nf * cap), dtype=torch.int64, device=dev)
        self.fields = torch.zeros(1 + nf * world * cap, dtype=torch.int64, device=dev)  # [count, field 0, ...]
        self.out = torch.zeros(max(plan.n_out, 1), dtype=torch.int64, device=dev)
        self.count = torch.zeros(1, dtype=torch.int64, device=dev)
        rel, _, _ = plan.scan_span(rank) if plan.off is not None else (np.zeros(1, np.int64), 0, 0)
        self.off = torch.from_numpy(np.ascontiguousarray(rel, dtype=np.int64)).to(dev)
        if torch.device(dev).type == "cuda":
            torch.cuda.synchronize(dev)

    @classmethod
    def from_host(cls, plan, rank, x, y, exchange=None, backend=None, device=None, nan=False, x_on_device=True):
        """Upload only this rank's element span of y (and of x, unless
        x_on_device=False: then only the candidates' x values are read from
        the host array, once per step) to its GPU."""
        import torch

        y = as_value_series(y)
        x = as_index_series(x, length(y))
        e0, e1 = plan.spans[rank] if plan.spans else (0, 0)
        dev = getattr(backend, "torch_device", None) or torch.device("cuda", backend.device if device is None
                                                                      else device)
        def put(a):
            a = a[e0:e1]
            if dev.type != "cuda":  # CPU test doubles
                return torch.from_numpy(np.ascontiguousarray(a))
            t = torch.empty(a.shape[0], dtype=_torch_dtype(a.dtype), device=dev)
            if a.shape[0]:
                _lib.upload(backend.ctx, t, np.ascontiguousarray(a))
            return t

        ys = put(y)
        xs = put(x) if plan.x_used and x is not None and x_on_device else None
        dts = (CODE[y.dtype], CODE[x.dtype] if x is not None else 0)
        return cls(plan, rank, ys, xs, exchange, backend, nan, dts, x_host=None if x_on_device else x)

    def _fill_x_bits(self):
        import torch

        self.backend.synchronize()
        cap = self.plan.cap
        cnt = int(self.rec[0].item())
        idx = self.rec[1 : 1 + cnt].cpu().numpy()
        v = np.ascontiguousarray(self.x_host[idx])
        bits = v.view({1: np.uint8, 2: np.uint16, 4: np.uint32, 8: np.uint64}[v.dtype.itemsize]).astype(np.uint64)
        self.rec[1 + cap : 1 + cap + cnt].copy_(torch.from_numpy(bits.view(np.int64)))
        if self.rec.is_cuda:
            torch.cuda.synchronize(self.rec.device)

    def step(self):
        p = self.plan
        self.backend.shard_record(p, self.rank, self.y, self.ydt, self.x, self.xdt, self.off, self.rec, self.nan)
        if self.x_host is not None and p.algo == "minmaxlttb":
            self._fill_x_bits()
        self.exchange.allgather(self.rec, self.recv)
        ld = p.world * p.cap
        if p.algo in WIDTH:
            self.backend.concat(self.recv, p.world, p.cap, 1, self.out, ld, self.count)
            return
        # MinMaxLTTB: fields = [m, full[ld], xbits[ld], ybits[ld]]
        self.backend.concat(self.recv, p.world, p.cap, 3, self.fields[1:], ld, self.fields[:1])
        xbits = self.fields[1 + ld : 1 + 2 * ld] if p.x_used else None
        ybits = self.fields[1 + 2 * ld : 1 + 3 * ld]
        self.backend.stage2(p, self.fields, xbits, self.xdt, ybits, self.ydt, self.out, self.count)

    def result(self):
        self.backend.synchronize()
        m = int(self.count.item())
        return self.out[:m].cpu().numpy().view(np.uint64)


def sharded_downsample(algo, *args, n_out, minmax_ratio=4, nan=False, group=None, device=None, backend=None,
                       exchange=None):
    """Sharded ``downsample(algo, [x,] y, n_out=...)``: every rank passes the
    same host series, uploads only its shard, and gets the full result
    (uint64, identical on all ranks, equal to the single-GPU / reference one)."""
    import torch.distributed as dist

    if len(args) == 1:
        x, y = None, args[0]
    elif len(args) == 2:
        x, y = args
    else:
        raise TypeError("expected positional arguments ([x,] y)")
    y = as_value_series(y)
    x = as_index_series(x, length(y))
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    plan = make_plan(algo, x, length(y), n_out, minmax_ratio, world)
    if plan.algo == "identity":
        return np.arange(plan.n, dtype=np.uint64)
    if plan.algo == "lttb":  # replicas only: the walk is sequential
        from . import algorithms

        return algorithms.lttb(x, y, n_out)
    if backend is None:
        backend = GpuBackend(rank if device is None else device)
    if exchange is None:
        exchange = default_exchange(backend.ctx, group)
    s = ShardedSeries.from_host(plan, rank, x, y, exchange, backend, nan=nan, x_on_device=False)
    s.step()
    return s.result()


class ShardedBatch:
    """Rank `rank`'s rows [s0, s1) of an S x L batch (contiguous chunks of
    ceil(S / world)), device-resident.  ``step()`` runs the batched MinMax on
    the rank's rows into a padded block [counts | indices] and all-gathers
    the blocks; ``result()`` returns (idx[S, n_out] uint64, counts[S])."""

    def __init__(self, S, L, n_out, rank, world, rows_dev, ydt, exchange, backend, nan=False):
        import torch

        self.S, self.L, self.n_out, self.rank, self.world, self.nan = S, L, n_out, rank, world, nan
        self.chunks = shard_ranges(S, world)
        self.rows = max(1, max(b - a for a, b in self.chunks))
        s0, s1 = self.chunks[rank]
        self.nrows = s1 - s0
        self.y, self.ydt = rows_dev, ydt
        self.exchange, self.backend = exchange, backend
        dev = rows_dev.device
        self.blk = torch.zeros(self.rows * (n_out + 1), dtype=torch.int64, device=dev)
        self.recv = torch.zeros(world * self.blk.numel(), dtype=torch.int64, device=dev)
        if torch.device(dev).type == "cuda":
            torch.cuda.synchronize(dev)

    def step(self):
        self.backend.batched_block(self.y, self.ydt, self.nrows, self.L, self.n_out, self.nan, self.blk, self.rows)
        self.exchange.allgather(self.blk, self.recv)

    def result(self):
        self.backend.synchronize()
        flat = self.recv.cpu().numpy().reshape(self.world, -1)
        idx = np.zeros((self.S, self.n_out), np.int64)
        counts = np.zeros(self.S, np.int64)
        for r, (a, b) in enumerate(self.chunks):
            k = b - a
            if k <= 0:
                continue
            counts[a:b] = flat[r, :k]
            idx[a:b] = flat[r, self.rows : self.rows + k * self.n_out].reshape(k, self.n_out)
        return idx.view(np.uint64), counts


def sharded_minmax_batched(Y, n_out, nan=False, group=None, device=None, backend=None, exchange=None):
    """Batched MinMax with the series partitioned across ranks: every rank
    passes the same host batch, uploads only its rows and gets the full
    (idx[S, n_out] uint64, counts[S]) -- row s equals minmax(Y[s])."""
    import torch
    import torch.distributed as dist

    Y = np.asarray(Y)
    if Y.dtype not in CODE:
        raise ValueError("unsupported dtype")
    if Y.ndim != 2:
        raise ValueError("expected a 2-D batch")
    if n_out < 2:
        raise ValueError("invalid n_out")
    if n_out % 2:
        raise ValueError("n_out must be a multiple of 2")
    S, L = Y.shape
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    if backend is None:
        backend = GpuBackend(rank if device is None else device)
    if exchange is None:
        exchange = default_exchange(backend.ctx, group)
    s0, s1 = shard_ranges(S, world)[rank]
    dev = getattr(backend, "torch_device", None) or torch.device("cuda", backend.device)
    rows = torch.from_numpy(np.ascontiguousarray(Y[s0:s1])).to(dev)
    b = ShardedBatch(S, L, n_out, rank, world, rows, CODE[Y.dtype], exchange, backend, nan)
    if L <= n_out:
        idx = np.zeros((S, n_out), np.int64)
        idx[:, :L] = np.arange(L)
        return idx.view(np.uint64), np.full(S, L, np.int64)
    b.step()
    return b.result()
