"""Multi-process (world_size 2, gloo on CPU) tests of the sharding layer.

paper_2307_05389_b200.distributed plans the shards (bin ranges, element
spans, frame points, record capacity), moves per-rank records through an
exchange and concatenates them in rank order; MinMaxLTTB feeds the gathered
candidates (with their raw x / y bits) to the triangle stage.  Here the
per-rank device work is a CPU test double built on the pinned oracle
(OracleBackend: the same record layout as include/tsds.h), so what is under
test is the product's plan, record, exchange and ordering logic; results
must equal the unsharded reference result exactly.
"""

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


_NP = {0: np.float16, 1: np.float32, 2: np.float64, 3: np.int8, 4: np.int16, 5: np.int32, 6: np.int64, 7: np.uint8,
       8: np.uint16, 9: np.uint32, 10: np.uint64}


def _bits(a):
    """Raw element bits zero-extended to int64 (the record's x / y fields)."""
    a = np.ascontiguousarray(a)
    u = a.view({1: np.uint8, 2: np.uint16, 4: np.uint32, 8: np.uint64}[a.dtype.itemsize])
    return u.astype(np.uint64).view(np.int64)


def _unbits(b, code):
    dt = np.dtype(_NP[code])
    u = np.asarray(b, np.int64).view(np.uint64).astype({1: np.uint8, 2: np.uint16, 4: np.uint32, 8: np.uint64}[dt.itemsize])
    return u.view(dt)


class OracleBackend:
    """CPU stand-in for GpuBackend (same signatures, same record layout)."""

    def __init__(self):
        import torch

        self.torch_device = torch.device("cpu")
        self.device = -1

    def _picks(self, plan, y, off, nan, width):
        from oracle import oracle as O

        nb = off.shape[0] - 1
        idx = np.zeros(width * max(nb, 1), np.int64)
        cnt = np.zeros(max(nb, 1), np.int64)
        O.bins_slots(width, y, off, 0, nb, idx, cnt, nan=nan)
        return O.compact_bins(idx, cnt[:nb], width)

    def shard_record(self, plan, rank, y_dev, ydt, x_dev, xdt, off_dev, rec, nan):
        from paper_2307_05389_b200.distributed import WIDTH

        b0, b1 = plan.ranges[rank]
        e0 = plan.spans[rank][0]
        y = y_dev.numpy()
        off = off_dev.numpy()
        r = np.zeros(rec.numel(), np.int64)
        cap = plan.cap
        if plan.algo in WIDTH:
            if b1 > b0:
                sel = self._picks(plan, y, off, nan, WIDTH[plan.algo]) + e0
                r[0] = sel.shape[0]
                r[1 : 1 + sel.shape[0]] = sel
        else:
            sel = self._picks(plan, y, off, nan, 2) + e0 if b1 > b0 else np.zeros(0, np.int64)
            if rank == 0:
                sel = np.concatenate([[0], sel])
            if rank == plan.world - 1:
                sel = np.concatenate([sel, [plan.n - 1]])
            sel = sel.astype(np.int64)
            k = sel.shape[0]
            r[0] = k
            r[1 : 1 + k] = sel
            if x_dev is not None:
                r[1 + cap : 1 + cap + k] = _bits(x_dev.numpy()[sel - e0])
            r[1 + 2 * cap : 1 + 2 * cap + k] = _bits(y[sel - e0])
        rec.copy_(__import__("torch").from_numpy(r))

    def concat(self, recv, world, cap, nf, out, ld_out, count):
        import torch

        recs = recv.numpy().reshape(world, 1 + nf * cap)
        parts = [[recs[r, 1 + f * cap : 1 + f * cap + recs[r, 0]] for r in range(world)] for f in range(nf)]
        total = sum(int(recs[r, 0]) for r in range(world))
        o = out.numpy()
        for f in range(nf):
            o[f * ld_out : f * ld_out + total] = np.concatenate(parts[f]) if total else []
        count.copy_(torch.tensor([total]))

    def stage2(self, plan, cand, xbits, xdt, ybits, ydt, out, count):
        import torch

        from oracle import oracle as O

        c = cand.numpy()
        m = int(c[0])
        full = c[1 : 1 + m].copy()
        if m <= plan.n_out:
            res = full
        else:
            y2 = _unbits(ybits.numpy()[:m], ydt)
            nb = plan.n_out - 2
            if xbits is None:
                off2 = (np.arange(nb + 1, dtype=np.int64) * (m - 2)) // nb + 1
                sel = O.lttb_walk(full, y2, off2)
            else:
                x2 = _unbits(xbits.numpy()[:m], xdt)
                off2 = O.equal_width(x2[1:-1], nb).astype(np.int64) + 1
                sel = O.lttb_walk(x2, y2, off2)
            res = full[sel]
        out.numpy()[: res.shape[0]] = res
        count.copy_(torch.tensor([res.shape[0]]))

    def batched_block(self, y_dev, ydt, nrows, L, n_out, nan, blk, rows):
        from oracle import oracle as O

        b = np.zeros(blk.numel(), np.int64)
        if nrows:
            idx, cnt = O.minmax_batched(y_dev.numpy(), n_out, nan=nan)
            b[:nrows] = cnt
            b[rows : rows + nrows * n_out] = idx.view(np.int64).reshape(-1)
        blk.copy_(__import__("torch").from_numpy(b))

    def synchronize(self):
        pass


def _worker(rank, world, port, cases, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_2307_05389_b200 import distributed as D
    from test_distributed_cpu import OracleBackend

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = []
        be = OracleBackend()
        for algo, x, y, n_out, kw in cases:
            args = (y,) if x is None else (x, y)
            got = D.sharded_downsample(algo, *args, n_out=n_out, backend=be, exchange=D.TorchExchange(), **kw)
            res.append(got.tolist())
        Y = np.stack([y for _, _, y, _, _ in cases[:1]] * 5)
        idx, cnt = D.sharded_minmax_batched(Y, 40, backend=be, exchange=D.TorchExchange())
        res.append((idx.tolist(), cnt.tolist()))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def _cases():
    import workloads as W

    cases = []
    y = W.random_series("f32", 20_003, 5, ties=True)
    x = W.random_x(20_003, 6, gaps=True)
    for algo, n_out in (("minmax", 100), ("m4", 100), ("minmaxlttb", 60)):
        cases.append((algo, None, y, n_out, {}))
        cases.append((algo, x, y, n_out, {}))
    xf = np.cumsum(np.random.default_rng(3).exponential(1.0, 20_003)).astype(np.float32)
    cases.append(("minmaxlttb", xf, y.astype(np.float16), 50, {"minmax_ratio": 3}))
    cases.append(("minmaxlttb", np.arange(20_003, dtype=np.int64) * 7, y, 60, {}))  # uniform x dropped
    yn = W.nan_series("f64", 9_001, 7, frac=0.01, at_starts=[0])
    cases.append(("m4", None, yn, 40, {"nan": True}))
    cases.append(("minmax", None, yn, 40, {}))
    cases.append(("minmaxlttb", None, yn, 30, {"minmax_ratio": 2}))
    cases.append(("minmax", None, y[:30], 40, {}))  # identity
    cases.append(("minmax", None, y, 2, {}))  # one bin: rank 1 has no bins
    cases.append(("minmaxlttb", None, y[:2000], 3, {"minmax_ratio": 8}))  # one sub-bin ... the last rank has none
    return cases


def test_sharded_equals_unsharded_world2():
    sys.path.insert(0, ROOT)
    from oracle import oracle as O

    cases = _cases()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cases, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[0] == out[1]
    for i, (algo, x, yy, n_out, kw) in enumerate(cases):
        args = (yy,) if x is None else (x, yy)
        kw2 = dict(kw)
        nan = kw2.pop("nan", False)
        want = O.downsample(algo, *args, n_out=n_out, nan=nan, **kw2)
        assert out[0][i] == want.tolist(), (i, algo, n_out, kw)
    idx, cnt = out[0][-1]
    want, wcnt = O.minmax_batched(np.stack([cases[0][2]] * 5), 40)
    assert cnt == wcnt.tolist()
    assert idx == want.tolist()


def test_shard_ranges_partition():
    sys.path.insert(0, ROOT)
    from paper_2307_05389_b200.distributed import shard_ranges

    for nb in (1, 2, 7, 1000, 9996):
        for world in (1, 2, 3, 8):
            r = shard_ranges(nb, world)
            assert len(r) == world
            assert r[0][0] == 0 and r[-1][1] == nb
            for (a, b), (c, d) in zip(r, r[1:]):
                assert b == c and a <= b


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_plan_spans_cover_every_bin_and_frame(world):
    """Every rank's element span holds its bins; ranks 0 / world-1 hold the
    MinMaxLTTB frame points; records are large enough for the worst rank."""
    sys.path.insert(0, ROOT)
    import workloads as W
    from paper_2307_05389_b200.distributed import make_plan

    x = W.random_x(50_000, 9, gaps=True)
    for algo, n_out in (("minmax", 400), ("m4", 400), ("minmaxlttb", 100)):
        for xx in (None, x):
            p = make_plan(algo, xx, 50_000, n_out, 4, world)
            assert len(p.ranges) == world == len(p.spans)
            for r, ((b0, b1), (e0, e1)) in enumerate(zip(p.ranges, p.spans)):
                if b1 > b0:
                    assert e0 <= p.off[b0] and p.off[b1] <= e1
                    per_bin = 2 if algo == "minmaxlttb" else {"minmax": 2, "m4": 4}[algo]
                    assert per_bin * (b1 - b0) + (2 if algo == "minmaxlttb" else 0) <= p.cap
            if algo == "minmaxlttb":
                assert p.spans[0][0] == 0 and p.spans[-1][1] == 50_000
